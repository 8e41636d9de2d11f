"""Helpers shared by the GPU parity tests: run the CUDA path through the C ABI and
the oracle on the same seeded inputs, and compare (tolerances from north_star)."""
from __future__ import annotations

import numpy as np
import torch

import lina_inputs as li
from oracle import moe

TOL = {"f32": 1e-5, "bf16": 2e-2}


def tdtype(dtype: str):
    return torch.float32 if dtype == "f32" else torch.bfloat16


def to_dev(a, dtype=None, device="cuda"):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(device)


def gpu_layer(cfg: li.LayerConfig, n_chunks: int, X, Wg, W1, W2, dY=None, capacity=None,
              override=None, comm=None, poison=False):
    """Run forward (+ backward when dY is given) of one rank at P=1 through the C ABI.
    poison: fill the saved and workspace buffers with 0xFF bytes (NaN in fp32 and bf16)
    first, so any read of a byte the layer did not write shows up in the results."""
    import paper_2210_17223_b200 as lina
    comm = comm or lina.Comm(1, 0, 0)
    C = cfg.capacity() if capacity is None else capacity
    dt = tdtype(cfg.dtype)
    layer = lina.MoELayer(comm, X.shape[0], cfg.d_model, cfg.d_ffn, cfg.num_experts, cfg.k, C, n_chunks, dt)
    if poison:
        layer.saved.fill_(0xFF)
        layer.workspace.fill_(0xFF)
    x = to_dev(X, dt); wg = to_dev(Wg, torch.float32); w1 = to_dev(W1, dt); w2 = to_dev(W2, dt)
    if override is not None:
        layer.route_t["idx"].copy_(to_dev(override[0].astype(np.int32)))
        layer.route_t["gate"].copy_(to_dev(override[1].astype(np.float32)))
    y = layer.forward(x, wg, w1, w2, want_route=True, override_routing=override is not None)
    out = {"y": y, **{k: v.clone() for k, v in layer.route_t.items()}}
    if dY is not None:
        dy = to_dev(dY, dt)
        dx, dwg, dw1, dw2 = layer.backward(dy, x, wg, w1, w2)
        out.update(dx=dx, dwg=dwg, dw1=dw1, dw2=dw2)
    torch.cuda.synchronize()
    return {k: v.float().cpu().numpy() if v.is_floating_point() else v.cpu().numpy() for k, v in out.items()}


def oracle_layer(cfg: li.LayerConfig, X, Wg, W1, W2, dY=None, capacity=None):
    C = cfg.capacity() if capacity is None else capacity
    fw = moe.moe_forward([X], Wg, W1, W2, cfg.k, C, cfg.dtype)
    out = {"fw": fw[0]}
    if dY is not None:
        out["bw"] = moe.moe_backward(fw, [X], [dY], Wg, W1, W2, cfg.k, cfg.dtype)
    return out


def assert_close(got, ref, tol, what):
    err = moe.normwise_error(got, ref)
    assert err <= tol, f"{what}: normwise error {err:.3e} > {tol:.1e}"
    return err


def compare(cfg, g, o, check_bwd=True, p_rtol=2e-6):
    """p_rtol bounds the fp32 probabilities and gate weights.  On grid inputs the logits are
    exact on both sides, so 2e-6 (a few ulp of the softmax) holds; on non-grid inputs the
    GPU's fp32 logits differ from the oracle's fp64-then-rounded ones by accumulation order
    (|dL| ~ 1e-6 |L|), which a softmax ratio amplifies by |L| — those callers pass 2e-5."""
    fw = o["fw"]
    assert np.array_equal(g["idx"], fw.idx), "routing idx differs"
    assert np.array_equal(g["slot"], fw.slot), "capacity slots differ"
    assert np.array_equal(g["counts"], fw.counts), "per-expert counts differ"
    assert np.allclose(g["gate"], fw.gate, rtol=p_rtol, atol=1e-7), \
        f"gate weights differ (max rel {np.max(np.abs(g['gate'] - fw.gate) / np.maximum(np.abs(fw.gate), 1e-30)):.2e})"
    assert np.allclose(g["probs"], fw.p, rtol=p_rtol, atol=1e-7), "probabilities differ"
    tol = TOL[cfg.dtype]
    errs = {"y": assert_close(g["y"], fw.y, tol, "y")}
    if check_bwd and "bw" in o:
        bw = o["bw"]
        errs["dx"] = assert_close(g["dx"], bw.dXs[0], tol, "dX")
        errs["dwg"] = assert_close(g["dwg"], bw.dWg, tol, "dWg")
        errs["dw1"] = assert_close(g["dw1"], bw.dW1, tol, "dW1")
        errs["dw2"] = assert_close(g["dw2"], bw.dW2, tol, "dW2")
    return errs
