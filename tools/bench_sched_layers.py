"""Allreduce scheduling across a multi-layer backward (S9 and its ablations, R23).

The paper's scheduling figures (fig:schedule_baseline / naive / optimal) are
about a step with several MoE layers: the non-expert gradients of block i become ready
when block i's backward ends, and their allreduce then competes with block i-1's
all-to-all.  One MoE layer (tools/bench_c3.py) has no next all-to-all to block, so the
NAIVE and DEFER ablations cannot show their cost there.  This tool chains `--layers` MoE
layers (C3 shape): forward y_i = layer_i(y_{i-1}); backward in reverse with dY of layer
i-1 = dX of layer i; after each layer's backward, `--grads` fp32 tensors of `--grad-mb` MB
(the block's attention / dense gradients) are handed to the scheduler.  It reports, per
policy, the device time of the whole backward and of the last allreduce, max over ranks.

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/bench_sched_layers.py
"""
from __future__ import annotations

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
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--grads", type=int, default=2)
    ap.add_argument("--grad-mb", type=float, default=16.8)
    ap.add_argument("--partition-mb", type=float, default=30.0)
    ap.add_argument("--n-chunks", type=int, default=1)
    ap.add_argument("--reps", type=int, default=8)
    ap.add_argument("--policies", default="NONE,BASELINE,LINA,NAIVE,DEFER")
    a = ap.parse_args()
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2210_17223_b200 as lina
    from paper_2210_17223_b200.lina import (LINA_SCHED_BASELINE, LINA_SCHED_DEFER, LINA_SCHED_LINA,
                                             LINA_SCHED_NAIVE)
    policies = {"NONE": None, "BASELINE": LINA_SCHED_BASELINE, "LINA": LINA_SCHED_LINA,
                "NAIVE": LINA_SCHED_NAIVE, "DEFER": LINA_SCHED_DEFER}

    cfg = li.with_tokens(li.CONFIGS[a.config], a.tokens)
    E, El = cfg.num_experts, cfg.num_experts // world
    uid = [lina.lina_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = lina.Comm(world, rank, local, uid[0], 8)
    dt = torch.bfloat16
    Wg, W1, W2 = li.layer_weights(cfg, 3, "balanced", experts=range(rank * El, (rank + 1) * El))
    X, dY = li.layer_tokens(cfg, 3, rank, "balanced")
    wg = torch.from_numpy(Wg).to(dev)
    w1 = torch.from_numpy(W1).to(dt).to(dev)
    w2 = torch.from_numpy(W2).to(dt).to(dev)
    x0 = torch.from_numpy(X).to(dt).to(dev)
    dy0 = torch.from_numpy(dY).to(dt).to(dev)
    layers = [lina.MoELayer(comm, cfg.tokens_per_rank, cfg.d_model, cfg.d_ffn, E, cfg.k, cfg.capacity(),
                            a.n_chunks, dt, dev) for _ in range(a.layers)]
    xs = [x0] + [torch.empty_like(x0) for _ in range(a.layers)]
    dxs = [torch.empty_like(x0) for _ in range(a.layers)]
    n_el = int(a.grad_mb * 2 ** 20 / 4)
    grads = [[torch.randn(n_el, device=dev) for _ in range(a.grads)] for _ in range(a.layers)]
    stream = torch.cuda.current_stream()
    ready = torch.cuda.Stream(dev)

    def step(policy):
        for i, layer in enumerate(layers):
            layer.forward(xs[i], wg, w1, w2, out=xs[i + 1])
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        dy = dy0
        for i in reversed(range(a.layers)):
            layers[i].backward(dy, xs[i], wg, w1, w2, dtokens=dxs[i])
            dy = dxs[i]
            if policy is not None:  # block i's non-expert gradients are ready now
                ev = torch.cuda.Event()
                ev.record(stream)
                ready.wait_event(ev)
                for g in grads[i]:
                    lina.lina_allreduce_submit(comm, g, ready)
        e1.record(stream)
        if policy is not None:
            lina.lina_allreduce_wait(comm, stream)
        e2.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), e0.elapsed_time(e2)

    res = {"world": world, "config": cfg.name, "tokens_per_rank": cfg.tokens_per_rank, "layers": a.layers,
           "grads_per_layer": f"{a.grads} x {a.grad_mb} MB fp32", "partition_mb": a.partition_mb,
           "n_chunks": a.n_chunks, "transport": os.environ.get("LINA_TRANSPORT", "fused")}
    for name in a.policies.split(","):
        pol = policies[name]
        if pol is not None:
            lina.lina_sched_config(comm, pol, int(a.partition_mb * 2 ** 20))
        ts = [step(pol) for _ in range(a.reps + 2)][2:]
        t = torch.tensor([sorted(v[0] for v in ts)[len(ts) // 2], sorted(v[1] for v in ts)[len(ts) // 2]],
                         dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name] = {"bwd_ms": float(t[0]), "ar_done_ms": float(t[1])}
    if rank == 0:
        base = res.get("NONE", {}).get("bwd_ms")
        if base:
            for name in a.policies.split(","):
                res[name]["bwd_slowdown"] = res[name]["bwd_ms"] / base
        print(json.dumps(res), flush=True)
    del layers
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
