"""C4 inference measurement: forward latency of the MoE layer
with the static placement (E/N experts per device) vs Lina's popularity-driven
replication (Eq. (1) + FFD from this batch's histogram), Zipf-skewed
synthetic tokens (s in {0.5, 1.0, 1.2}).  Device time per forward, max over ranks,
p50/p95 over the iterations; max/mean routed tokens per device for both placements
(from the top-1 histogram of the batch).

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        --master-port 29541 tools/bench_c4.py [--iters 50]"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import lina_inputs as li  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--zipf", default="0,0.5,1.0,1.2", help="Zipf exponents; 0 = uniform popularity (the balanced ideal)")
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--batches", type=int, default=5, help="distinct seeded batches cycled over the iterations")
    ap.add_argument("--modes", default="static,replicated")
    a = ap.parse_args()
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2210_17223_b200 as lina
    from paper_2210_17223_b200.lina import PlacementTables

    cfg = li.CONFIGS["C4"]
    E, T, d = cfg.num_experts, cfg.tokens_per_rank, cfg.d_model
    El = E // world
    mpd = 2 * El  # twice the static experts per device
    uid = [lina.lina_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = lina.Comm(world, rank, local, uid[0], 8)
    dt = torch.bfloat16
    Wg, W1, W2 = li.layer_weights(cfg, 11, "zipf")
    wg = torch.from_numpy(Wg).to(dev)
    w1 = torch.from_numpy(W1).to(dt).to(dev)
    w2 = torch.from_numpy(W2).to(dt).to(dev)
    desc = lina.make_desc(T, d, cfg.d_ffn, E, cfg.k, T, 1, dt)
    ws = torch.empty(lina.lina_moe_infer_workspace_size(comm, desc, mpd), dtype=torch.uint8, device=dev)
    out = torch.empty((T, d), dtype=dt, device=dev)
    static = PlacementTables([1] * E, [[e // El] for e in range(E)],
                             [list(range(dv * El, (dv + 1) * El)) for dv in range(world)])
    stream = torch.cuda.current_stream()
    for s in [float(v) for v in a.zipf.split(",")]:
        # the expert directions come from the weight seed; batches differ by their token stream id
        xs = [torch.from_numpy(li.layer_tokens(cfg, 11, rank + world * b, "zipf", zipf_s=s)[0]).to(dt).to(dev)
              for b in range(a.batches)]
        # global top-1 histogram of batch 0 (input statistics for the balance numbers)
        cnt = torch.bincount((xs[0].float() @ wg).argmax(1), minlength=E).to(torch.int64)
        dist.all_reduce(cnt)
        res = {"world": world, "config": cfg.name, "tokens_per_rank": T, "zipf_s": s, "max_per_device": mpd}
        for name, pl in (("static", static), ("replicated", None)):
            if name not in a.modes.split(","):
                continue
            plan = None
            ts = []
            for it in range(a.iters + 3):
                x = xs[it % a.batches]
                dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                p = lina.lina_moe_infer_forward(comm, desc, x, wg, w1, w2, out, ws, placement=pl, max_per_device=mpd,
                                                want_plan=(it == 0))
                e1.record(stream)
                torch.cuda.synchronize()
                if it == 0:
                    plan = p
                if it >= 3:
                    ts.append(e0.elapsed_time(e1))
            t = torch.tensor(ts, dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t = np.sort(t.cpu().numpy())
            tab = static if pl is not None else plan
            per_dev = np.zeros(world)
            c = cnt.cpu().numpy().astype(np.float64)
            for e in range(E):
                for dv in tab.replica_device[e]:
                    per_dev[dv] += c[e] / len(tab.replica_device[e])
            res[name] = {"fwd_ms_p50": float(t[len(t) // 2]), "fwd_ms_p95": float(t[int(0.95 * (len(t) - 1))]),
                         "max_over_mean_tokens": float(per_dev.max() / per_dev.mean()),
                         "replicas": list(tab.replicas) if pl is None else None,
                         "hosted_per_device": [len(h) for h in tab.hosted]}
        if rank == 0:
            print(json.dumps(res), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
