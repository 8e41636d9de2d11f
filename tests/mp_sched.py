"""Micro-op allreduce scheduler (S9) under torch.distributed.run, one rank per GPU.

Each rank runs the MoE layer backward while four synthetic non-expert gradients
(BERT-large-attention-sized, 4 x 16.8 MB fp32) are queued for the
DP allreduce, once with the BASELINE policy (whole tensors issued at once, sharing the
links with the all-to-all) and once with LINA (equal micro-ops admitted
only while no all-to-all is queued or in flight).
Checks: the allreduced gradients equal torch.distributed's sum (both policies) and
dWg allreduced through the scheduler equals the sum of the ranks' dWg; reports the
backward time, the backward all-to-all time and the allreduce completion time.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29531 tests/mp_sched.py --config C3 --tokens 2048
"""
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
    ap.add_argument("--tokens", type=int, default=2048)
    ap.add_argument("--n-chunks", type=int, default=4)
    ap.add_argument("--partition-mb", type=float, default=4.0)
    ap.add_argument("--grad-mb", type=float, default=16.8)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2210_17223_b200 as lina
    from paper_2210_17223_b200.lina import (LINA_SCHED_BASELINE, LINA_SCHED_DEFER, LINA_SCHED_LINA,
                                             LINA_SCHED_NAIVE)

    cfg = li.with_tokens(li.CONFIGS[a.config], a.tokens)
    E, El = cfg.num_experts, cfg.num_experts // world
    uid = [lina.lina_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = lina.Comm(world, rank, local, uid[0], 8)
    Wg, W1, W2 = li.layer_weights(cfg, 3, "balanced", experts=range(rank * El, (rank + 1) * El))
    X, dY = li.layer_tokens(cfg, 3, rank, "balanced")
    dt = torch.bfloat16
    layer = lina.MoELayer(comm, cfg.tokens_per_rank, cfg.d_model, cfg.d_ffn, E, cfg.k, cfg.capacity(),
                          a.n_chunks, dt, dev)
    x = torch.from_numpy(X).to(dt).to(dev)
    dy = torch.from_numpy(dY).to(dt).to(dev)
    wg = torch.from_numpy(Wg).to(dev)
    w1 = torch.from_numpy(W1).to(dt).to(dev)
    w2 = torch.from_numpy(W2).to(dt).to(dev)
    n_el = int(a.grad_mb * 2 ** 20 / 4)
    g0 = torch.Generator(device=dev).manual_seed(100 + rank)
    base_grads = [torch.randn(n_el, device=dev, generator=g0) for _ in range(4)]
    expect = [g.clone() for g in base_grads]
    for e in expect:
        dist.all_reduce(e)
    stream = torch.cuda.current_stream()
    results = {}
    ok = True
    for name, pol in (("BASELINE", LINA_SCHED_BASELINE), ("LINA", LINA_SCHED_LINA),
                      ("NAIVE", LINA_SCHED_NAIVE), ("DEFER", LINA_SCHED_DEFER)):
        lina.lina_sched_config(comm, pol, int(a.partition_mb * 2 ** 20))
        times = []
        for rep in range(a.reps + 1):
            grads = [g.clone() for g in base_grads]
            layer.forward(x, wg, w1, w2)
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            for g in grads:  # non-expert gradients become ready as the MoE backward starts
                lina.lina_allreduce_submit(comm, g, stream)
            dx, dwg, dw1, dw2 = layer.backward(dy, x, wg, w1, w2)
            e1.record(stream)
            lina.lina_allreduce_submit(comm, dwg, stream)
            lina.lina_allreduce_wait(comm, stream)
            e2.record(stream)
            torch.cuda.synchronize()
            if rep > 0:
                times.append((e0.elapsed_time(e1), e0.elapsed_time(e2)))
            for g, ref in zip(grads, expect):
                ok &= bool(torch.allclose(g, ref, rtol=1e-5, atol=1e-4))
            dwg_ref = torch.empty_like(dwg)
            # dwg was allreduced in place by the scheduler: compare with an independent sum
            layer.forward(x, wg, w1, w2)
            _, dwg_local, _, _ = layer.backward(dy, x, wg, w1, w2)
            dwg_ref.copy_(dwg_local)
            dist.all_reduce(dwg_ref)
            ok &= bool(torch.allclose(dwg, dwg_ref, rtol=1e-4, atol=1e-5))
        issued, deferred = lina.lina_sched_stats(comm)
        bwd = sorted(t[0] for t in times)[len(times) // 2]
        ar = sorted(t[1] for t in times)[len(times) // 2]
        results[name] = {"bwd_ms_median": bwd, "ar_done_ms_median": ar, "microops_issued": issued,
                         "deferred_polls": deferred}
    gathered = [None] * world
    dist.gather_object((ok, results), gathered if rank == 0 else None, dst=0)
    if rank == 0:
        allok = all(g[0] for g in gathered)
        print("MP_SCHED", "OK" if allok else "FAIL", json.dumps({"world": world, "config": cfg.name,
              "tokens": cfg.tokens_per_rank, "n_chunks": a.n_chunks, "partition_mb": a.partition_mb,
              "rank0": gathered[0][1]}), flush=True)
        ok = allok
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.broadcast(flag, 0)
    comm.close()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
