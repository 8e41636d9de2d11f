"""Multi-rank parity of the expert-parallel layer (run under torch.distributed.run, one
rank per GPU).  Every rank runs forward+backward through lina_comm (NCCL all-to-all
micro-ops); rank 0 gathers every rank's outputs and gradients and compares them with
the oracle, which simulates all ranks in one process.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29511 tests/mp_parity.py --config C2 --tokens 512 --n-chunks 2
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
    ap.add_argument("--config", default="C2")
    ap.add_argument("--tokens", type=int, default=512)
    ap.add_argument("--n-chunks", type=int, default=2)
    ap.add_argument("--experts", type=int, default=0)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--seed", type=int, default=77)
    ap.add_argument("--check-chunks", type=int, default=0, help="also run with this n_chunks and compare bitwise")
    ap.add_argument("--poison", action="store_true", help="start from NaN-filled saved/workspace buffers")
    ap.add_argument("--graph", action="store_true",
                    help="also capture fwd+bwd in a CUDA graph, replay it 3 times, require bitwise equal results")
    ap.add_argument("--interleave", action="store_true",
                    help="run a second layer B between A's forward and backward (fwd A, fwd B, bwd B, "
                         "bwd A) on the same communicator; A must still match the oracle")
    ap.add_argument("--shared-ws", action="store_true",
                    help="with --interleave: layer B uses layer A's workspace (scratch may be shared between "
                         "layers on one communicator; lina.h)")
    ap.add_argument("--dropless", action="store_true",
                    help="capacity 0: the dropless layout (count exchange + unequal split, §8(f) row 4); "
                         "the oracle runs with C = T (no drops)")
    ap.add_argument("--pack", type=int, default=1,
                    help="expert packing factor m (P:376): groups of m ranks host the same m*E/world experts")
    ap.add_argument("--pack-exchange", action="store_true",
                    help="build the packed weights with lina_pack_weights from the unpacked ones (P:505)")
    ap.add_argument("--ragged-ranks", type=int, default=0,
                    help="rank r holds T - r*R tokens (same capacity C on every rank): the peer-visible buffer "
                         "regions must not depend on num_tokens")
    ap.add_argument("--shared-gpu", action="store_true",
                    help="every rank on GPU 0 with a host-bootstrap communicator (no NCCL; tests/mp_util.py)")
    a = ap.parse_args()
    from tests.mp_util import setup
    world, rank, dev, comm, flag_dev = setup(a.shared_gpu, 0)
    import paper_2210_17223_b200 as lina

    changes = {}
    if a.experts:
        changes["num_experts"] = a.experts
    if a.k:
        changes["k"] = a.k
    cfg = li.with_tokens(li.CONFIGS[a.config], a.tokens, **changes)
    E, El = cfg.num_experts, cfg.num_experts // world
    m = max(1, a.pack)
    G = rank // m                    # packing group; its experts [G*m*El, (G+1)*m*El)
    hosted = range(G * m * El, (G + 1) * m * El)
    Wg, W1, W2 = li.layer_weights(cfg, a.seed, experts=hosted)
    exchange_ok = True
    if a.pack_exchange and m > 1:
        _, W1u, W2u = li.layer_weights(cfg, a.seed, experts=range(rank * El, (rank + 1) * El))
        tdt_ = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
        got = []
        for Wu in (W1u, W2u):
            src = torch.from_numpy(Wu).to(tdt_).to(dev)
            dst = torch.full((m * El,) + tuple(Wu.shape[1:]), float("nan"), dtype=tdt_, device=dev)
            lina.lina_pack_weights(comm, E, 1, m, src, dst)
            got.append(dst.float().cpu().numpy())
        exchange_ok = np.array_equal(got[0], torch.from_numpy(W1).to(tdt_).float().numpy()) and \
            np.array_equal(got[1], torch.from_numpy(W2).to(tdt_).float().numpy())
    def T_of(r):
        return cfg.tokens_per_rank - r * a.ragged_ranks

    X, dY = li.layer_tokens(cfg, a.seed, rank, num_tokens=T_of(rank))
    tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32

    C_layer = 0 if a.dropless else cfg.capacity()

    def run(n_chunks):
        layer = lina.MoELayer(comm, T_of(rank), cfg.d_model, cfg.d_ffn, E, cfg.k, C_layer,
                              n_chunks, tdt, dev, pack=m)
        if a.poison:  # every byte the layer reads must be one it (or a peer) wrote this step
            layer.saved.fill_(0xFF)
            layer.workspace.fill_(0xFF)
            torch.cuda.synchronize()
            dist.barrier()
        x = torch.from_numpy(X).to(tdt).to(dev)
        wg = torch.from_numpy(Wg).to(dev)
        w1 = torch.from_numpy(W1).to(tdt).to(dev)
        w2 = torch.from_numpy(W2).to(tdt).to(dev)
        dy = torch.from_numpy(dY).to(tdt).to(dev)
        y = layer.forward(x, wg, w1, w2, want_route=True)
        finite_b = True
        if a.interleave:  # layer B's exchanges run between A's forward and backward
            layer_b = lina.MoELayer(comm, T_of(rank), cfg.d_model, cfg.d_ffn, E, cfg.k, C_layer,
                                    n_chunks, tdt, dev, pack=m)
            if a.shared_ws:
                layer_b.workspace = layer.workspace
            XB, dYB = li.layer_tokens(cfg, a.seed + 1, rank, num_tokens=T_of(rank))
            xb = torch.from_numpy(XB).to(tdt).to(dev)
            yb = layer_b.forward(xb, wg, w1, w2)
            dxb = layer_b.backward(torch.from_numpy(dYB).to(tdt).to(dev), xb, wg, w1, w2)[0]
            finite_b = bool(torch.isfinite(yb).all()) and bool(torch.isfinite(dxb).all())
        dx, dwg, dw1, dw2 = layer.backward(dy, x, wg, w1, w2)
        torch.cuda.synchronize()
        comm.check()
        out = {"y": y.float().cpu().numpy(), "dx": dx.float().cpu().numpy(), "dwg": dwg.cpu().numpy(),
               "dw1": dw1.float().cpu().numpy(), "dw2": dw2.float().cpu().numpy(),
               "idx": layer.route_t["idx"].cpu().numpy(), "slot": layer.route_t["slot"].cpu().numpy(),
               "finite_b": finite_b, "exchange_ok": exchange_ok}
        if a.graph:  # replays must be full steps: the cross-rank rounds live in device memory
            gy, gdx = torch.empty_like(y), torch.empty_like(dx)
            gdwg, gdw1, gdw2 = torch.empty_like(dwg), torch.empty_like(dw1), torch.empty_like(dw2)
            cap = torch.cuda.Stream(dev)
            cap.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            dist.barrier()
            with torch.cuda.graph(g, stream=cap):
                layer.forward(x, wg, w1, w2, out=gy)
                layer.backward(dy, x, wg, w1, w2, gdx, gdwg, gdw1, gdw2)
            torch.cuda.synchronize()
            dist.barrier()
            for _ in range(3):
                for t in (gy, gdx, gdw1, gdw2):
                    t.fill_(float("nan"))
                g.replay()
                torch.cuda.synchronize()
                comm.check()
                same = all(torch.equal(u, v) for u, v in ((gy, y), (gdx, dx), (gdwg, dwg), (gdw1, dw1), (gdw2, dw2)))
                if not same:
                    out["graph_mismatch"] = True
        return out

    res = run(a.n_chunks)
    gathered = [None] * world
    dist.gather_object(res, gathered if rank == 0 else None, dst=0)
    ok = True
    if rank == 0 and not all(g["finite_b"] for g in gathered):
        print("interleaved layer B produced non-finite values", flush=True)
        ok = False
    if rank == 0 and any(g.get("graph_mismatch") for g in gathered):
        print("CUDA graph replay differs from the eager step", flush=True)
        ok = False
    if a.check_chunks:
        res2 = run(a.check_chunks)
        # outputs and token gradients are bitwise chunk-invariant (each row's arithmetic is
        # fixed); the weight gradients reduce over rows in chunk-dependent 64-row K blocks on
        # the tensor cores, so they agree to accumulation rounding only
        from oracle import moe as _m
        same = all(np.array_equal(res[k], res2[k]) for k in ("y", "dx", "idx", "slot")) and \
            all(_m.normwise_error(res2[k], res[k]) <= 1e-2 for k in ("dw1", "dw2", "dwg"))
        flags = [None] * world
        dist.gather_object(same, flags if rank == 0 else None, dst=0)
        if rank == 0 and not all(flags):
            print(f"chunk invariance FAILED: n={a.n_chunks} vs n={a.check_chunks}", flush=True)
            ok = False
    if rank == 0:
        from oracle import moe
        Wg_all, W1_all, W2_all = li.layer_weights(cfg, a.seed)
        Xs = [li.layer_tokens(cfg, a.seed, r, num_tokens=T_of(r))[0] for r in range(world)]
        dYs = [li.layer_tokens(cfg, a.seed, r, num_tokens=T_of(r))[1] for r in range(world)]
        C_ref = cfg.tokens_per_rank if a.dropless else cfg.capacity()
        fw = moe.moe_forward(Xs, Wg_all, W1_all, W2_all, cfg.k, C_ref, cfg.dtype)
        bw = moe.moe_backward(fw, Xs, dYs, Wg_all, W1_all, W2_all, cfg.k, cfg.dtype)
        tol = 1e-5 if cfg.dtype == "f32" else 2e-2
        dwg_sum = sum(g["dwg"] for g in gathered)   # the DP allreduce of R12
        errs = {}
        for r in range(world):
            g = gathered[r]
            ok &= np.array_equal(g["idx"], fw[r].idx) and np.array_equal(g["slot"], fw[r].slot)
            errs[f"y{r}"] = moe.normwise_error(g["y"], fw[r].y)
            errs[f"dx{r}"] = moe.normwise_error(g["dx"], bw.dXs[r])
            lo, hi = (r // m) * m * El, (r // m + 1) * m * El   # the experts rank r hosts
            errs[f"dw1_{r}"] = moe.normwise_error(g["dw1"], bw.dW1[lo:hi])
            errs[f"dw2_{r}"] = moe.normwise_error(g["dw2"], bw.dW2[lo:hi])
        errs["dwg"] = moe.normwise_error(dwg_sum, bw.dWg)
        ok &= all(v <= tol for v in errs.values())
        ok &= all(g["exchange_ok"] for g in gathered)
        print("MP_PARITY", "OK" if ok else "FAIL", f"world={world} cfg={cfg.name} T={cfg.tokens_per_rank} "
              f"n={a.n_chunks}" + (" dropless" if a.dropless else "") + (f" pack={m}" if m > 1 else ""), " ".join(f"{k}={v:.2e}" for k, v in errs.items()), flush=True)
    flag = torch.tensor([1 if ok else 0], device=flag_dev)
    dist.broadcast(flag, 0)
    comm.close()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
