"""C3 contention measurement: the MoE layer backward with four
concurrent non-expert gradient allreduces (4 x 16.8 MB fp32, ready when the backward
starts), scheduled BASELINE (whole tensors at once) vs LINA (micro-ops admitted only
while no all-to-all is queued or in flight), plus the
backward alone.  The gradients' ready event is the backward's start; they are handed
to the scheduler while the backward runs (as the layers above the MoE layer finish
theirs).  Device time, median over reps, max over ranks.

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        --master-port 29531 tools/bench_c3.py [--tokens 8192] [--chunks 1,4] [--partitions 4,16,30]
Prints one JSON line per (n_chunks, partition) on rank 0."""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import lina_inputs as li  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--chunks", default="1,4")
    ap.add_argument("--partitions", default="4,16,30")
    ap.add_argument("--grad-mb", type=float, default=16.8)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--policies", default="BASELINE,LINA,NAIVE,DEFER",
                    help="schedulers to compare (NAIVE / DEFER are the paper's ablations, R23)")
    a = ap.parse_args()
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2210_17223_b200 as lina
    from paper_2210_17223_b200.lina import (LINA_SCHED_BASELINE, LINA_SCHED_DEFER, LINA_SCHED_LINA,
                                             LINA_SCHED_NAIVE)
    policies = {"BASELINE": LINA_SCHED_BASELINE, "LINA": LINA_SCHED_LINA, "NAIVE": LINA_SCHED_NAIVE,
                "DEFER": LINA_SCHED_DEFER}

    cfg = li.with_tokens(li.CONFIGS[a.config], a.tokens)
    E, El = cfg.num_experts, cfg.num_experts // world
    uid = [lina.lina_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = lina.Comm(world, rank, local, uid[0], 8)
    Wg, W1, W2 = li.layer_weights(cfg, 3, "balanced", experts=range(rank * El, (rank + 1) * El))
    X, dY = li.layer_tokens(cfg, 3, rank, "balanced")
    dt = torch.bfloat16
    x = torch.from_numpy(X).to(dt).to(dev)
    dy = torch.from_numpy(dY).to(dt).to(dev)
    wg = torch.from_numpy(Wg).to(dev)
    w1 = torch.from_numpy(W1).to(dt).to(dev)
    w2 = torch.from_numpy(W2).to(dt).to(dev)
    n_el = int(a.grad_mb * 2 ** 20 / 4)
    grads = [torch.randn(n_el, device=dev) for _ in range(4)]
    stream = torch.cuda.current_stream()
    ready = torch.cuda.Stream(dev)

    def run(layer, policy):
        """median (bwd ms, AR-done ms) over reps; policy None = no allreduce."""
        ts = []
        for rep in range(a.reps + 2):
            layer.forward(x, wg, w1, w2)
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            ready.wait_event(e0)  # the gradients are ready when the MoE backward starts ...
            layer.backward(dy, x, wg, w1, w2)
            e1.record(stream)
            if policy is not None:  # ... and handed to the scheduler while it runs
                for g in grads:
                    lina.lina_allreduce_submit(comm, g, ready)
            if policy is not None:
                lina.lina_allreduce_wait(comm, stream)
            e2.record(stream)
            torch.cuda.synchronize()
            if rep >= 2:
                ts.append((e0.elapsed_time(e1), e0.elapsed_time(e2)))
        t = torch.tensor([sorted(v[0] for v in ts)[len(ts) // 2], sorted(v[1] for v in ts)[len(ts) // 2]],
                         dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0]), float(t[1])

    for n in [int(v) for v in a.chunks.split(",")]:
        layer = lina.MoELayer(comm, cfg.tokens_per_rank, cfg.d_model, cfg.d_ffn, E, cfg.k, cfg.capacity(), n, dt,
                              dev)
        alone, _ = run(layer, None)
        for part in [float(v) for v in a.partitions.split(",")]:
            res = {"world": world, "config": cfg.name, "tokens_per_rank": cfg.tokens_per_rank, "n_chunks": n,
                   "partition_mb": part, "grads": f"4 x {a.grad_mb} MB fp32", "bwd_alone_ms": alone,
                   "transport": os.environ.get("LINA_TRANSPORT", "fused")}
            for name in a.policies.split(","):
                pol = policies[name]
                lina.lina_sched_config(comm, pol, int(part * 2 ** 20))
                bwd, done = run(layer, pol)
                res[name] = {"bwd_ms": bwd, "bwd_slowdown": bwd / alone, "ar_done_ms": done}
            if rank == 0:
                print(json.dumps(res), flush=True)
        del layer
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
