"""Multi-rank inference with popularity-driven replication (S10), one rank per GPU:
the plan equals the oracle's placement of the global histogram; the replicated
layer's outputs equal (bitwise) the outputs with the static one-expert-set-per-device
placement (P9) and match the oracle; per-device received-token counts follow the
replica split (R14).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29521 tests/mp_infer.py --tokens 512 --zipf 1.0
"""
import argparse
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
    ap.add_argument("--tokens", type=int, default=512)
    ap.add_argument("--zipf", type=float, default=1.0)
    ap.add_argument("--experts", type=int, default=0)
    ap.add_argument("--mpd", type=int, default=0, help="max experts per device (0 = 2 E/N)")
    ap.add_argument("--seed", type=int, default=11)
    ap.add_argument("--min-replicas", type=int, default=1,
                    help="fail unless the plan replicates some expert at least this many times")
    ap.add_argument("--shared-gpu", action="store_true",
                    help="every rank on GPU 0 with a host-bootstrap communicator (no NCCL; tests/mp_util.py)")
    a = ap.parse_args()
    from tests.mp_util import setup
    world, rank, dev, comm, flag_dev = setup(a.shared_gpu, 8)
    import paper_2210_17223_b200 as lina
    from paper_2210_17223_b200.lina import PlacementTables

    changes = {"num_experts": a.experts} if a.experts else {}
    cfg = li.with_tokens(li.CONFIGS["C4"], a.tokens, **changes)
    E, T = cfg.num_experts, cfg.tokens_per_rank
    mpd = a.mpd or 2 * E // world
    Wg, W1, W2 = li.layer_weights(cfg, a.seed, "zipf")
    X, _ = li.layer_tokens(cfg, a.seed, rank, "zipf", zipf_s=a.zipf)
    dt = torch.bfloat16
    x = torch.from_numpy(X).to(dt).to(dev)
    wg = torch.from_numpy(Wg).to(dev)
    w1 = torch.from_numpy(W1).to(dt).to(dev)
    w2 = torch.from_numpy(W2).to(dt).to(dev)
    desc = lina.make_desc(T, cfg.d_model, cfg.d_ffn, E, cfg.k, T, 1, dt)
    ws = torch.empty(lina.lina_moe_infer_workspace_size(comm, desc, mpd), dtype=torch.uint8, device=dev)

    def run(placement):
        out = torch.empty((T, cfg.d_model), dtype=dt, device=dev)
        plan = lina.lina_moe_infer_forward(comm, desc, x, wg, w1, w2, out, ws, placement=placement,
                                           max_per_device=mpd)
        torch.cuda.synchronize()
        comm.check()
        return out.float().cpu().numpy(), plan

    y_rep, plan = run(None)
    rows_rep = lina.lina_infer_last_rows(comm)  # (received per source, sent per device) under the plan
    El = E // world
    static = PlacementTables([1] * E, [[e // El] for e in range(E)],
                             [list(range(dv * El, (dv + 1) * El)) for dv in range(world)])
    y_sta, _ = run(static)
    rows_sta = lina.lina_infer_last_rows(comm)
    res = {"y_rep": y_rep, "y_sta": y_sta, "plan": (plan.replicas, plan.replica_device, plan.hosted),
           "rows_rep": rows_rep, "rows_sta": rows_sta}
    gathered = [None] * world
    dist.gather_object(res, gathered if rank == 0 else None, dst=0)
    ok = True
    if rank == 0:
        from oracle import moe
        from oracle import placement as oplace
        Xs = [li.layer_tokens(cfg, a.seed, r, "zipf", zipf_s=a.zipf)[0] for r in range(world)]
        fw = moe.moe_forward(Xs, Wg, W1, W2, cfg.k, T, cfg.dtype)
        counts = np.stack([f.counts for f in fw])
        pop = counts.sum(0) / counts.sum()
        ref = oplace.place(list(pop), world, mpd)
        plan_ok = all(g["plan"] == (ref["replicas"], ref["replica_device"], ref["hosted"]) for g in gathered)
        bitwise = all(np.array_equal(g["y_rep"], g["y_sta"]) for g in gathered)
        errs = [moe.normwise_error(gathered[r]["y_rep"], fw[r].y) for r in range(world)]
        # balance: tokens per device under the plan vs static
        send = oplace.route_counts(counts, ref, world)
        per_dev = np.array(send).sum(axis=(0, 2))
        static_dev = counts.sum(0).reshape(world, El).sum(1)
        # rows each device received from each source = the oracle's replica split (R14), under
        # the replicated plan and under the static placement; and what each rank sent
        sta_ref = {"replicas": [1] * E, "replica_device": [[e // El] for e in range(E)]}
        send_sta = oplace.route_counts(counts, sta_ref, world)
        rows_ok = True
        for dv in range(world):
            for key, snd in (("rows_rep", send), ("rows_sta", send_sta)):
                recv, sent = gathered[dv][key]
                rows_ok &= recv == [int(sum(snd[s][dv])) for s in range(world)]
                rows_ok &= sent == [int(sum(snd[dv][o])) for o in range(world)]
        max_r = max(ref["replicas"])
        repl_ok = max_r >= a.min_replicas
        ok = plan_ok and bitwise and max(errs) <= 2e-2 and rows_ok and repl_ok
        print("MP_INFER", "OK" if ok else "FAIL", f"world={world} E={E} T={T} zipf={a.zipf} mpd={mpd}",
              f"plan_ok={plan_ok} bitwise={bitwise} rows_ok={rows_ok} max_replicas={max_r} "
              f"(need >= {a.min_replicas}) err={max(errs):.2e} replicas={ref['replicas']}",
              f"rows received by each device from each source: "
              f"{[gathered[dv]['rows_rep'][0] for dv in range(world)]}",
              f"max/mean tokens per device: replicated {per_dev.max() / per_dev.mean():.2f} "
              f"static {static_dev.max() / static_dev.mean():.2f}", flush=True)
    flag = torch.tensor([1 if ok else 0], device=flag_dev)
    dist.broadcast(flag, 0)
    comm.close()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
