"""configs[1] at full size on every rank, in the launch configuration bench.py times
(fused transport, n_chunks = 1, one CUDA-graph replay per step), one rank per GPU:
routing bit-exact on every token of every rank; y and dX on sampled tokens of every rank
computed one by one with the oracle (the expert of each kept assignment may live on any
rank).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29541 tests/mp_fullsize.py
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
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--samples", type=int, default=32)
    a = ap.parse_args()
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2210_17223_b200 as lina
    from oracle import moe

    cfg = li.CONFIGS[a.config]
    E, El, T, d, k, C = cfg.num_experts, cfg.num_experts // world, cfg.tokens_per_rank, cfg.d_model, cfg.k, \
        cfg.capacity()
    uid = [lina.lina_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = lina.Comm(world, rank, local, uid[0], 8)
    Wg, W1, W2 = li.layer_weights(cfg, a.seed, "grid")          # all experts (oracle side)
    X, dY = li.layer_tokens(cfg, a.seed, rank, "grid")
    dt = torch.bfloat16
    x = torch.from_numpy(X).to(dt).to(dev)
    dy = torch.from_numpy(dY).to(dt).to(dev)
    wg = torch.from_numpy(Wg).to(dev)
    w1 = torch.from_numpy(W1[rank * El:(rank + 1) * El]).to(dt).to(dev)
    w2 = torch.from_numpy(W2[rank * El:(rank + 1) * El]).to(dt).to(dev)
    layer = lina.MoELayer(comm, T, d, cfg.d_ffn, E, k, C, 1, dt, dev)
    layer.saved.fill_(0xFF)
    layer.workspace.fill_(0xFF)
    y = torch.empty((T, d), dtype=dt, device=dev)
    dx = torch.empty_like(y)
    dwg, dw1, dw2 = torch.empty_like(wg), torch.empty_like(w1), torch.empty_like(w2)
    layer.forward(x, wg, w1, w2, out=y, want_route=True)         # eager step (routing outputs)
    layer.backward(dy, x, wg, w1, w2, dx, dwg, dw1, dw2)
    torch.cuda.synchronize()
    route = {kk: v.cpu().numpy() for kk, v in layer.route_t.items()}
    cap = torch.cuda.Stream(dev)
    cap.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    dist.barrier()
    with torch.cuda.graph(g, stream=cap):
        layer.forward(x, wg, w1, w2, out=y)
        layer.backward(dy, x, wg, w1, w2, dx, dwg, dw1, dw2)
    torch.cuda.synchronize()
    dist.barrier()
    for _ in range(2):                                         # the bench's launch mode
        y.fill_(float("nan"))
        dx.fill_(float("nan"))
        g.replay()
    torch.cuda.synchronize()
    comm.check()
    Y = y.float().cpu().numpy()
    DX = dx.float().cpu().numpy()

    # ---- oracle side: routing of this rank's tokens on every token, experts on samples
    L = moe.gate_logits(X, Wg)
    p = moe.softmax(L)
    idx = moe.top_k(L, k)
    gate = moe.gate_weights(p, idx)
    slot, counts = moe.capacity_slots(idx, E, C)
    ok = bool(np.array_equal(route["idx"], idx) and np.array_equal(route["slot"], slot)
              and np.array_equal(route["counts"], counts))
    rng = np.random.default_rng(100 + rank)
    sample = np.concatenate([[0, T - 1], rng.choice(T - 1, a.samples - 2, replace=False) + 1])
    rf = moe.RankForward(L=L[sample], p=p[sample], idx=idx[sample], gate=gate[sample], slot=slot[sample],
                         counts=counts, y=np.zeros((len(sample), d)))
    for n, t in enumerate(sample):
        for j in range(k):
            if slot[t, j] >= 0:
                e = idx[t, j]
                h, o = moe.expert_ffn(X[t:t + 1], W1[e], W2[e], "bf16")
                rf.h[(n, j)] = h[0]
                rf.o[(n, j)] = o[0]
    rf.y = moe.combine(rf, k, "bf16")
    bw = moe.moe_backward([rf], [X[sample]], [dY[sample]], Wg, W1, W2, k, "bf16")
    ey = moe.normwise_error(Y[sample], rf.y)
    edx = moe.normwise_error(DX[sample], bw.dXs[0])
    ok = ok and ey <= 2e-2 and edx <= 2e-2 and np.isfinite(Y).all() and np.isfinite(DX).all()
    res = [None] * world
    dist.gather_object((ok, ey, edx), res if rank == 0 else None, dst=0)
    allok = True
    if rank == 0:
        allok = all(r[0] for r in res)
        print("MP_FULLSIZE", "OK" if allok else "FAIL", f"world={world} {cfg.name} T/rank={T} C={C}",
              " ".join(f"r{i}: y {r[1]:.2e} dX {r[2]:.2e}" for i, r in enumerate(res)), flush=True)
    flag = torch.tensor([1 if allok else 0], device=dev)
    dist.broadcast(flag, 0)
    comm.close()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
