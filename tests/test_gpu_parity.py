"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same
seeded inputs.  Routing (idx, slot, counts) must match bit-exactly; outputs and
gradients within the north_star tolerances (fp32 1e-5, bf16 2e-2, normwise)."""
import numpy as np
import pytest
import torch

import lina_inputs as li
from oracle import moe
from tests.parity_util import TOL, compare, gpu_layer, oracle_layer, to_dev, tdtype

pytestmark = pytest.mark.gpu


def _case(name, tokens=None, seed=1234, family="grid", **changes):
    cfg = li.CONFIGS[name]
    if tokens is not None or changes:
        cfg = li.with_tokens(cfg, tokens or cfg.tokens_per_rank, **changes)
    Wg, W1, W2 = li.layer_weights(cfg, seed, family)
    X, dY = li.layer_tokens(cfg, seed, 0, family)
    return cfg, X, Wg, W1, W2, dY


@pytest.mark.parametrize("n_chunks", [1, 4])
def test_c1_full_fwd_bwd(n_chunks):
    """configs[0] at full size: fp32, 4 experts, top-1, capacity factor 1.0 (drops occur)."""
    cfg, X, Wg, W1, W2, dY = _case("C1")
    g = gpu_layer(cfg, n_chunks, X, Wg, W1, W2, dY)
    o = oracle_layer(cfg, X, Wg, W1, W2, dY)
    assert (o["fw"].slot < 0).any()
    compare(cfg, g, o)


def test_c1_chunk_invariance_bitwise():
    """P8: n_chunks only re-slices the GEMMs; outputs and gradients are bitwise equal."""
    cfg, X, Wg, W1, W2, dY = _case("C1")
    a = gpu_layer(cfg, 1, X, Wg, W1, W2, dY)
    for n in (2, 4, 7):
        b = gpu_layer(cfg, n, X, Wg, W1, W2, dY)
        for key in ("y", "dx", "dwg", "dw1", "dw2", "idx", "slot"):
            assert np.array_equal(a[key], b[key]), (n, key)


@pytest.mark.parametrize("k,capacity", [(1, 512), (2, 128), (2, 1), (3, 300)])
def test_c1_variants(k, capacity):
    cfg, X, Wg, W1, W2, dY = _case("C1", k=k)
    g = gpu_layer(cfg, 2 if capacity > 1 else 1, X, Wg, W1, W2, dY, capacity=capacity)
    o = oracle_layer(cfg, X, Wg, W1, W2, dY, capacity=capacity)
    compare(cfg, g, o)


@pytest.mark.parametrize("tokens", [1, 63, 333])
def test_ragged_token_counts(tokens):
    cfg, X, Wg, W1, W2, dY = _case("C1", tokens=tokens, k=2)
    g = gpu_layer(cfg, 1, X, Wg, W1, W2, dY)
    o = oracle_layer(cfg, X, Wg, W1, W2, dY)
    compare(cfg, g, o)


@pytest.mark.parametrize("n_chunks", [1, 3])
def test_c2_reduced_bf16(n_chunks):
    """configs[1] shapes (E=8, top-2, d=768, f=3072, bf16) at 512 tokens."""
    cfg, X, Wg, W1, W2, dY = _case("C2", tokens=512)
    g = gpu_layer(cfg, n_chunks, X, Wg, W1, W2, dY)
    o = oracle_layer(cfg, X, Wg, W1, W2, dY)
    compare(cfg, g, o)


@pytest.mark.parametrize("n_chunks", [1, 3])
def test_c2_poisoned_workspace(n_chunks):
    """Saved state and workspace start as NaN bytes: the layer must only read what it wrote
    (padding rows it leaves unwritten, are never read as data)."""
    cfg, X, Wg, W1, W2, dY = _case("C2", tokens=512)
    g = gpu_layer(cfg, n_chunks, X, Wg, W1, W2, dY, poison=True)
    for k in ("y", "dx", "dwg", "dw1", "dw2"):
        assert np.isfinite(g[k]).all(), f"{k} has non-finite values"
    o = oracle_layer(cfg, X, Wg, W1, W2, dY)
    compare(cfg, g, o)


def test_c3_reduced_bf16():
    """configs[2] shapes (E=16, top-2, d=1024, f=4096, capacity 1.25) at 256 tokens."""
    cfg, X, Wg, W1, W2, dY = _case("C3", tokens=256)
    g = gpu_layer(cfg, 2, X, Wg, W1, W2, dY)
    o = oracle_layer(cfg, X, Wg, W1, W2, dY)
    compare(cfg, g, o)


def test_c5_reduced_bf16_forward():
    """configs[4] shapes (E=64, top-2, d=2048, f=8192) at 128 tokens: forward parity."""
    cfg, X, Wg, W1, W2, dY = _case("C5", tokens=128)
    g = gpu_layer(cfg, 1, X, Wg, W1, W2)
    o = oracle_layer(cfg, X, Wg, W1, W2)
    compare(cfg, g, o, check_bwd=False)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_identity_experts_roundtrip(dtype):
    """P5 on the GPU: combine(dispatch(x)) = x · Σ_kept g within one ulp of dtype."""
    cfg, X, Wg, _, _, _ = _case("C1", tokens=300, k=2, dtype=dtype)
    d, f, E = cfg.d_model, cfg.d_ffn, cfg.num_experts
    W1 = np.zeros((E, f, d), np.float32); W2 = np.zeros((E, d, f), np.float32)
    for e in range(E):
        W1[e, :d] = np.eye(d); W1[e, d:2 * d] = -np.eye(d)
        W2[e, :, :d] = np.eye(d); W2[e, :, d:2 * d] = -np.eye(d)
    g = gpu_layer(cfg, 2, X, Wg, W1, W2)
    gsum = (g["gate"] * (g["slot"] >= 0)).sum(1, keepdims=True).astype(np.float64)
    ref = X.astype(np.float64) * gsum
    ulp = 2.0 ** -8 if dtype == "bf16" else 2.0 ** -23
    assert np.all(np.abs(g["y"] - ref) <= ulp * np.abs(ref) + 1e-30)
    assert (g["slot"] < 0).any()


def test_override_routing_non_grid_inputs():
    """Non-grid (balanced) inputs: routing is fed from the oracle so the FFN/combine/backward
    arithmetic is compared on identical assignments."""
    cfg, X, Wg, W1, W2, dY = _case("C2", tokens=256, family="balanced")
    o = oracle_layer(cfg, X, Wg, W1, W2, dY)
    g = gpu_layer(cfg, 2, X, Wg, W1, W2, dY, override=(o["fw"].idx, o["fw"].gate))
    tol = TOL["bf16"]
    from tests.parity_util import assert_close
    assert np.array_equal(g["slot"], o["fw"].slot)
    assert_close(g["y"], o["fw"].y, tol, "y")
    assert_close(g["dw1"], o["bw"].dW1, tol, "dW1")
    assert_close(g["dw2"], o["bw"].dW2, tol, "dW2")


def test_c2_full_size_sampled():
    """configs[1] at full size (8192 tokens, the bench launch configuration, n_chunks=1):
    routing bit-exact on every token; y and dX on a sample of tokens computed one by one."""
    cfg, X, Wg, W1, W2, dY = _case("C2")
    g = gpu_layer(cfg, 1, X, Wg, W1, W2, dY)
    L = moe.gate_logits(X, Wg)
    p = moe.softmax(L)
    idx = moe.top_k(L, cfg.k)
    gate = moe.gate_weights(p, idx)
    slot, counts = moe.capacity_slots(idx, cfg.num_experts, cfg.capacity())
    assert np.array_equal(g["idx"], idx)
    assert np.array_equal(g["slot"], slot)
    assert np.array_equal(g["counts"], counts)
    rng = np.random.default_rng(0)
    sample = np.concatenate([[0, cfg.tokens_per_rank - 1], rng.choice(cfg.tokens_per_rank - 1, 62, replace=False) + 1])
    Xs, dYs = X[sample], dY[sample]
    rf = moe.RankForward(L=L[sample], p=p[sample], idx=idx[sample], gate=gate[sample], slot=slot[sample],
                         counts=counts, y=np.zeros((len(sample), cfg.d_model)))
    for n, t in enumerate(sample):
        for j in range(cfg.k):
            if slot[t, j] >= 0:
                e = idx[t, j]
                h, o = moe.expert_ffn(X[t:t + 1], W1[e], W2[e], "bf16")
                rf.h[(n, j)] = h[0]
                rf.o[(n, j)] = o[0]
    rf.y = moe.combine(rf, cfg.k, "bf16")
    bw = moe.moe_backward([rf], [Xs], [dYs], Wg, W1, W2, cfg.k, "bf16")   # dX rows are per-token exact
    from tests.parity_util import assert_close
    assert_close(g["y"][sample], rf.y, TOL["bf16"], "y (sampled)")
    assert_close(g["dx"][sample], bw.dXs[0], TOL["bf16"], "dX (sampled)")


def test_c5_full_tokens_routing_and_sampled_rows():
    """configs[4]'s token count and gate (32768 tokens, d = 2048, E = 64, top-2, capacity 1.25)
    with d_ffn = 256 (the expert FFN shape does not touch routing; full C5 weights in fp64 would
    not fit the host): routing, slots and counts bit-exact on every token of the bench's
    gate launch (256 CTAs of 128 tokens, 2 per SM) and y, dX on a
    sample of tokens computed one by one."""
    cfg, X, Wg, W1, W2, dY = _case("C5", d_ffn=256)
    assert cfg.tokens_per_rank == 32768 and cfg.num_experts == 64
    g = gpu_layer(cfg, 1, X, Wg, W1, W2, dY)
    L = moe.gate_logits(X, Wg)
    p = moe.softmax(L)
    idx = moe.top_k(L, cfg.k)
    gate = moe.gate_weights(p, idx)
    slot, counts = moe.capacity_slots(idx, cfg.num_experts, cfg.capacity())
    assert np.array_equal(g["idx"], idx)
    assert np.array_equal(g["slot"], slot)
    assert np.array_equal(g["counts"], counts)
    assert np.allclose(g["gate"], gate, rtol=2e-6, atol=1e-7)
    rng = np.random.default_rng(1)
    T = cfg.tokens_per_rank
    sample = np.concatenate([[0, 127, 128, 255, 256, T - 1], rng.choice(T - 2, 26, replace=False) + 1])
    Xs, dYs = X[sample], dY[sample]
    rf = moe.RankForward(L=L[sample], p=p[sample], idx=idx[sample], gate=gate[sample], slot=slot[sample],
                         counts=counts, y=np.zeros((len(sample), cfg.d_model)))
    for n, t in enumerate(sample):
        for j in range(cfg.k):
            if slot[t, j] >= 0:
                e = idx[t, j]
                h, o = moe.expert_ffn(X[t:t + 1], W1[e], W2[e], "bf16")
                rf.h[(n, j)] = h[0]
                rf.o[(n, j)] = o[0]
    rf.y = moe.combine(rf, cfg.k, "bf16")
    bw = moe.moe_backward([rf], [Xs], [dYs], Wg, W1, W2, cfg.k, "bf16")
    from tests.parity_util import assert_close
    assert_close(g["y"][sample], rf.y, TOL["bf16"], "y (sampled)")
    assert_close(g["dx"][sample], bw.dXs[0], TOL["bf16"], "dX (sampled)")


def test_comm_and_errors():
    import paper_2210_17223_b200 as lina
    comm = lina.Comm(1, 0, 0)
    bad = lina.make_desc(10, 30, 64, 5, 9, -1, 40, "bf16")
    with pytest.raises(lina.LinaError) as ei:
        lina.lina_moe_workspace_size(comm, bad)
    msg = str(ei.value)
    for frag in ["k not in", "capacity < 0", "n_chunks", "d_model % 16"]:
        assert frag in msg, msg
    good = lina.make_desc(64, 64, 256, 4, 1, 16, 1, "f32")
    ws, sv = lina.lina_moe_workspace_size(comm, good)
    small = torch.empty(8, dtype=torch.uint8, device="cuda")
    x = torch.zeros(64, 64, device="cuda")
    with pytest.raises(lina.LinaError) as ei:
        lina.lina_moe_forward(comm, good, x, torch.zeros(64, 4, device="cuda"), torch.zeros(4, 256, 64, device="cuda"),
                              torch.zeros(4, 64, 256, device="cuda"), torch.empty_like(x),
                              torch.empty(sv, dtype=torch.uint8, device="cuda"), small)
    assert ei.value.status == 6
    comm.close()


@pytest.mark.parametrize("n_chunks", [1, 2])
def test_cuda_graph_replay_bitwise(n_chunks):
    """The layer is stream-ordered and host-sync free: a captured fwd+bwd replays as a
    full step (bench.py times replays), bitwise equal to the eager step."""
    import paper_2210_17223_b200 as lina
    cfg, X, Wg, W1, W2, dY = _case("C2", tokens=512)
    dt = tdtype(cfg.dtype)
    comm = lina.Comm(1, 0, 0)
    layer = lina.MoELayer(comm, X.shape[0], cfg.d_model, cfg.d_ffn, cfg.num_experts, cfg.k, cfg.capacity(),
                          n_chunks, dt)
    x, dy = to_dev(X, dt), to_dev(dY, dt)
    wg, w1, w2 = to_dev(Wg, torch.float32), to_dev(W1, dt), to_dev(W2, dt)
    y = layer.forward(x, wg, w1, w2)
    dx, dwg, dw1, dw2 = layer.backward(dy, x, wg, w1, w2)
    torch.cuda.synchronize()
    outs = [torch.empty_like(t) for t in (y, dx, dwg, dw1, dw2)]
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        layer.forward(x, wg, w1, w2, out=outs[0])
        layer.backward(dy, x, wg, w1, w2, *outs[1:])
    for _ in range(2):
        for t in outs:
            t.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        for got, ref in zip(outs, (y, dx, dwg, dw1, dw2)):
            assert torch.equal(got, ref)
    comm.close()


def test_two_layers_interleaved_fwd_fwd_bwd_bwd():
    """Two MoE layers on one communicator run as in a model step — forward A, forward B,
    backward B, backward A — each with its own saved state and workspace; every output
    and gradient equals the oracle's single-layer result for that layer's inputs."""
    import paper_2210_17223_b200 as lina
    cfg = li.with_tokens(li.CONFIGS["C2"], 512)
    Wg, W1, W2 = li.layer_weights(cfg, 5, "grid")
    XA, dYA = li.layer_tokens(cfg, 6, 0, "grid")
    XB, dYB = li.layer_tokens(cfg, 7, 0, "grid")
    comm = lina.Comm(1, 0, 0)
    dt = tdtype(cfg.dtype)
    wg, w1, w2 = to_dev(Wg, torch.float32), to_dev(W1, dt), to_dev(W2, dt)
    layers = {n: lina.MoELayer(comm, 512, cfg.d_model, cfg.d_ffn, cfg.num_experts, cfg.k, cfg.capacity(), 1, dt)
              for n in "AB"}
    x = {"A": to_dev(XA, dt), "B": to_dev(XB, dt)}
    dy = {"A": to_dev(dYA, dt), "B": to_dev(dYB, dt)}
    y = {n: layers[n].forward(x[n], wg, w1, w2) for n in "AB"}
    grads = {n: layers[n].backward(dy[n], x[n], wg, w1, w2) for n in "BA"}
    torch.cuda.synchronize()
    for n, X, dY in (("A", XA, dYA), ("B", XB, dYB)):
        o = oracle_layer(cfg, X, Wg, W1, W2, dY)
        tol = TOL[cfg.dtype]
        assert moe.normwise_error(y[n].float().cpu().numpy(), o["fw"].y) <= tol, n
        dx, dwg, dw1, dw2 = (t.float().cpu().numpy() for t in grads[n])
        assert moe.normwise_error(dx, o["bw"].dXs[0]) <= tol, n
        assert moe.normwise_error(dwg, o["bw"].dWg) <= tol, n
        assert moe.normwise_error(dw1, o["bw"].dW1) <= tol, n
        assert moe.normwise_error(dw2, o["bw"].dW2) <= tol, n


@pytest.mark.parametrize("tail,half", [("0", "1"), ("0", "0"), ("1", "0")])
def test_c5_shapes_fwd_bwd_two_cta_tiles(tail, half, monkeypatch):
    """configs[4] layer dims (d=2048, f=8192, top-2, capacity 1.25) with 16 experts at 1024
    tokens: 128 rows per expert segment (> 96), so the expert GEMMs run the 2-CTA 256-row
    tiles the C5 bench runs, with K = 8192 in GEMM2 / dgrad2 and M = 2048 / 8192 in the
    wgrads; forward and backward against the oracle, without and with the opt-in tail split
    (LINA_TAIL128=1: a segment's last <= 128 rows as single-CTA tiles in a second launch),
    and with / without the half tails (LINA_HALF128, default on: a segment's last <= 128
    rows as an M = 128 cta_group::2 tile in the same launch, the 2x2 TMEM layout).
    (All 64 experts at full C5 would need the oracle's fp64 weight gradients, 34 GB; the
    forward at E = 64 is the test above.)"""
    monkeypatch.setenv("LINA_TAIL128", tail)
    monkeypatch.setenv("LINA_HALF128", half)
    cfg, X, Wg, W1, W2, dY = _case("C5", tokens=1024, num_experts=16)
    assert cfg.tokens_per_rank * cfg.k / cfg.num_experts > 96
    g = gpu_layer(cfg, 1, X, Wg, W1, W2, dY)
    o = oracle_layer(cfg, X, Wg, W1, W2, dY)
    compare(cfg, g, o)


@pytest.mark.parametrize("experts,k,tokens", [(32, 2, 1024), (64, 2, 1000), (64, 3, 777), (24, 1, 640)])
def test_gate_backward_tensor_core(experts, k, tokens):
    """E > 16 on the bf16 path: dX and dWg go through the tcgen05 gate-backward kernels
    (gate_bwd_tc.cu: the persistent dX kernel fused with the gather of the k returned rows,
    the split-K dWg and the fp32 dL split into bf16 terms) — forward and backward against
    the oracle at C5's top-k / capacity with d = 512, f = 1024, ragged token counts
    (777, 1000: a last 128-token block partly empty) and k = 3 (the KM = 8 variant)."""
    cfg, X, Wg, W1, W2, dY = _case("C5", tokens=tokens, num_experts=experts, k=k, d_model=512, d_ffn=1024)
    g = gpu_layer(cfg, 1, X, Wg, W1, W2, dY)
    o = oracle_layer(cfg, X, Wg, W1, W2, dY)
    compare(cfg, g, o)


def test_c2_full_size_weight_gradients():
    """configs[1] at full size (8192 tokens, ~2048 rows per expert, the bench shape at N=1):
    y, dX, dWg and the expert weight gradients dW1, dW2 (K = 2048+ rows per wgrad) against
    the oracle over every element."""
    cfg, X, Wg, W1, W2, dY = _case("C2")
    g = gpu_layer(cfg, 1, X, Wg, W1, W2, dY)
    o = oracle_layer(cfg, X, Wg, W1, W2, dY)
    compare(cfg, g, o)


def test_c2_chunk_invariance_bf16():
    """P8 on the bf16 tensor-core path: y and dX are bitwise equal for every n_chunks (each
    row's arithmetic is fixed); dW1 / dW2 reduce rows in 64-row K blocks that follow the chunk
    boundaries, so they agree to accumulation rounding only."""
    cfg, X, Wg, W1, W2, dY = _case("C2", tokens=2048)
    a = gpu_layer(cfg, 1, X, Wg, W1, W2, dY)
    for n in (2, 4):
        b = gpu_layer(cfg, n, X, Wg, W1, W2, dY)
        for key in ("y", "dx", "dwg", "idx", "slot"):
            assert np.array_equal(a[key], b[key]), (n, key)
        for key in ("dw1", "dw2"):
            assert moe.normwise_error(b[key], a[key]) <= 1e-2, (n, key)


# ---------------------------------------------------------------- dropless layout (§8(f) row 4)


@pytest.mark.parametrize("name,tokens,k,dtype", [("C1", 512, 1, "f32"), ("C1", 333, 2, "f32"),
                                                 ("C2", 512, 2, "bf16"), ("C2", 63, 2, "bf16")])
def test_dropless_single_gpu(name, tokens, k, dtype):
    """capacity 0: no token is dropped; outputs and gradients equal the oracle with C = T."""
    cfg, X, Wg, W1, W2, dY = _case(name, tokens=tokens, k=k, dtype=dtype)
    g = gpu_layer(cfg, 1, X, Wg, W1, W2, dY, capacity=0, poison=True)
    o = oracle_layer(cfg, X, Wg, W1, W2, dY, capacity=tokens)
    assert (g["slot"] >= 0).all()
    compare(cfg, g, o)


def test_dropless_c5_shapes_two_cta():
    """configs[4] dims at 16 experts / 1024 tokens through the dropless layout (256-row tiles)."""
    cfg, X, Wg, W1, W2, dY = _case("C5", tokens=1024, num_experts=16)
    g = gpu_layer(cfg, 1, X, Wg, W1, W2, dY, capacity=0)
    o = oracle_layer(cfg, X, Wg, W1, W2, dY, capacity=1024)
    compare(cfg, g, o)


def test_dropless_skewed_routing():
    """Zipf-skewed routing (most tokens on a few experts, some experts empty): every row of the
    hot experts' long blocks is processed — the case capacity padding handles worst."""
    cfg = li.with_tokens(li.CONFIGS["C4"], 512, num_experts=8, k=2, d_model=256, d_ffn=512)
    Wg, W1, W2 = li.layer_weights(cfg, 5, "zipf")
    X, dY = li.layer_tokens(cfg, 5, 0, "zipf", zipf_s=1.5)
    g = gpu_layer(cfg, 1, X, Wg, W1, W2, dY, capacity=0)
    o = oracle_layer(cfg, X, Wg, W1, W2, dY, capacity=512)
    assert np.bincount(g["idx"][:, 0], minlength=8).max() > 512 * 0.3
    compare(cfg, g, o, p_rtol=2e-5)  # non-grid inputs (parity_util.compare)


def test_dropless_footprint_against_padded_layout():
    """The point of the dropless layout: saved + workspace bytes well below the C = T padding."""
    import paper_2210_17223_b200 as lina
    comm = lina.Comm(1, 0, 0)
    cfg = li.CONFIGS["C5"]
    T, E = cfg.tokens_per_rank, cfg.num_experts
    dl = lina.lina_moe_workspace_size(comm, lina.make_desc(T, cfg.d_model, cfg.d_ffn, E, cfg.k, 0, 1, torch.bfloat16))
    pad = lina.lina_moe_workspace_size(comm, lina.make_desc(T, cfg.d_model, cfg.d_ffn, E, cfg.k, T, 1, torch.bfloat16))
    cap = lina.lina_moe_workspace_size(comm, lina.make_desc(T, cfg.d_model, cfg.d_ffn, E, cfg.k, cfg.capacity(), 1,
                                                            torch.bfloat16))
    print(f"C5 saved+workspace GB: dropless {sum(dl) / 1e9:.2f}, C=T {sum(pad) / 1e9:.2f}, "
          f"C=1.25 {sum(cap) / 1e9:.2f}")
    assert sum(dl) * 8 < sum(pad)
