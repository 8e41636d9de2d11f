"""Expert packing end to end (§8(f) row 3): train steps of one MoE
layer on the variable layout, feed the packing controller the device-timed FFN and
all-to-all micro-op times of every step (max over ranks, so every rank decides the same),
and when it packs, exchange the expert parameters (lina_pack_weights) and continue with
desc.pack = m.  Prints one JSON line per step and checks the packed layer against the
unpacked one at the end (same routing, same math: y and dX equal, dW within 1e-2).

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        --master-port 29561 tools/pack_controller.py --config C2 --d-ffn 512
"""
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
    ap.add_argument("--config", default="C2")
    ap.add_argument("--tokens", type=int, default=0)
    ap.add_argument("--d-ffn", type=int, default=0, help="override d_ffn (small FFN: the all-to-all dominates)")
    ap.add_argument("--experts", type=int, default=0)
    ap.add_argument("--steps", type=int, default=24)
    ap.add_argument("--start", type=int, default=10)
    ap.add_argument("--every", type=int, default=4)
    ap.add_argument("--seed", type=int, default=5)
    a = ap.parse_args()
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2210_17223_b200 as lina

    changes = {}
    if a.d_ffn:
        changes["d_ffn"] = a.d_ffn
    if a.experts:
        changes["num_experts"] = a.experts
    base = li.CONFIGS[a.config]
    cfg = li.with_tokens(base, a.tokens or base.tokens_per_rank, **changes)
    T, d, f, E, k = cfg.tokens_per_rank, cfg.d_model, cfg.d_ffn, cfg.num_experts, cfg.k
    El = E // world
    uid = [lina.lina_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = lina.Comm(world, rank, local, uid[0])
    dt = torch.bfloat16
    Wg, W1, W2 = li.layer_weights(cfg, a.seed, "balanced", experts=range(rank * El, (rank + 1) * El))
    X, dY = li.layer_tokens(cfg, a.seed, rank, "balanced")
    x, dy = torch.from_numpy(X).to(dt).to(dev), torch.from_numpy(dY).to(dt).to(dev)
    wg = torch.from_numpy(Wg).to(dev)
    w1, w2 = torch.from_numpy(W1).to(dt).to(dev), torch.from_numpy(W2).to(dt).to(dev)
    w1_0, w2_0 = w1.clone(), w2.clone()  # the unpacked weights (final check)
    pack = 1
    layer = lina.MoELayer(comm, T, d, f, E, k, 0, 1, dt, dev, pack=pack)
    ctl = lina.PackController(world, a.start, a.every)
    log = []
    for step in range(1, a.steps + 1):
        lina.lina_profile_read(comm)
        lina.lina_profile_enable(comm, 1)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        layer.forward(x, wg, w1, w2)
        layer.backward(dy, x, wg, w1, w2)
        ev1.record()
        torch.cuda.synchronize()
        lina.lina_profile_enable(comm, 0)
        pr = lina.lina_profile_read(comm)
        # "the controller records the completion times of all-to-all and FFN micro-ops":
        # FFN = the expert-GEMM phases, all-to-all = the micro-op intervals (max over ranks)
        t = torch.tensor([pr["gemm_ms"], pr["a2a_op_ms"], ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ffn, a2a, step_ms = (float(v) for v in t)
        new_pack, changed = ctl.step(ffn, a2a)
        rec = {"step": step, "pack": pack, "ffn_ms": ffn, "a2a_ms": a2a, "step_ms": step_ms}
        if changed:  # one-time synchronous parameter exchange, then the packed layer
            rec["repack_to"] = new_pack
            nw1 = torch.empty((new_pack * El,) + tuple(w1.shape[1:]), dtype=dt, device=dev)
            nw2 = torch.empty((new_pack * El,) + tuple(w2.shape[1:]), dtype=dt, device=dev)
            lina.lina_pack_weights(comm, E, pack, new_pack, w1, nw1)
            lina.lina_pack_weights(comm, E, pack, new_pack, w2, nw2)
            w1, w2, pack = nw1, nw2, new_pack
            layer = lina.MoELayer(comm, T, d, f, E, k, 0, 1, dt, dev, pack=pack)
        log.append(rec)
        if rank == 0:
            print(json.dumps(rec), flush=True)
    # the packed layer computes what the unpacked one does
    ref = lina.MoELayer(comm, T, d, f, E, k, 0, 1, dt, dev, pack=1)
    y0 = ref.forward(x, wg, w1_0, w2_0)
    dx0, dwg0, dw10, _ = ref.backward(dy, x, wg, w1_0, w2_0)
    y1 = layer.forward(x, wg, w1, w2)
    dx1, dwg1, dw11, _ = layer.backward(dy, x, wg, w1, w2)
    torch.cuda.synchronize()
    G = rank // pack
    mine = slice((rank % pack) * El, (rank % pack + 1) * El) if pack > 1 else slice(0, El)
    same = bool(torch.equal(y0, y1)) and bool(torch.equal(dx0, dx1)) and bool(torch.equal(dwg0, dwg1))
    dw_err = float((dw11[mine].float() - dw10.float()).abs().max() / dw10.float().abs().max().clamp_min(1e-30))
    flag = torch.tensor([1 if (same and dw_err <= 1e-2) else 0], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps({"final_pack": pack, "group_of_rank0": G, "y_dx_dwg_bitwise": same, "dw1_err": dw_err,
                          "PACK_CONTROLLER": "OK" if flag.item() == 1 else "FAIL"}), flush=True)
    comm.close()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
