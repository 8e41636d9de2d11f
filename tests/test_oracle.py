"""Pins for the CPU oracle (runs without a GPU).

Every check below fixes the oracle against something other than itself:
integer arithmetic, closed forms, brute force, textbook special cases, library
routines from another package, central finite differences, or hand-derived
golden tables under tests/golden/ (each with its citation).
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

import lina_inputs as li
from oracle import moe, placement

# ---------------------------------------------------------------- rounding


def test_round_bf16_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(20000).astype(np.float32) * 7,
                        # exact ties: 9 significant bits with last bit set
                        (np.arange(256, 512, dtype=np.float32) * 2 + 1) / 1024])
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(moe.round_bf16(x.astype(np.float64)), ref)


# ---------------------------------------------------------------- gating


def test_logits_exact_against_integer_matmul():
    """P1: grid inputs are k/64, so 4096·L is an integer matmul, exact in int64."""
    rng = np.random.default_rng(1)
    T, d, E = 64, 768, 8
    Xi = rng.integers(-31, 32, size=(T, d))
    Wi = rng.integers(-31, 32, size=(d, E))
    L = moe.gate_logits(Xi / 64.0, Wi / 64.0)
    exact = (Xi.astype(np.int64) @ Wi.astype(np.int64)).astype(np.float64) / 4096.0
    assert np.array_equal(L, exact)


def test_softmax_closed_forms():
    E = 8
    L = np.full((3, E), 1.7)
    assert np.allclose(moe.softmax(L), 1.0 / E, rtol=0, atol=1e-7)
    L2 = np.array([[0.3, -1.1], [5.0, 5.0], [-2.0, 3.0]])
    p = moe.softmax(L2)
    sig = 1.0 / (1.0 + np.exp(-(L2[:, 0] - L2[:, 1])))
    assert np.allclose(p[:, 0], sig, rtol=1e-6, atol=0)
    assert np.allclose(p.sum(1), 1.0, atol=1e-6)


def _topk_by_rank_count(L, k):
    """Independent definition: expert e sits at position j iff exactly j experts beat it
    (higher logit, or equal logit and lower id)."""
    T, E = L.shape
    out = np.full((T, k), -1)
    for t in range(T):
        for e in range(E):
            beat = sum(1 for f in range(E) if L[t, f] > L[t, e] or (L[t, f] == L[t, e] and f < e))
            if beat < k:
                out[t, beat] = e
    return out


@pytest.mark.parametrize("k", [1, 2, 3])
def test_topk_brute_force_with_ties(k):
    rng = np.random.default_rng(2)
    T, d, E = 40, 16, 6
    X = li.grid(rng, (T, d))
    Wg = li.grid(rng, (d, E))
    Wg[:, 3] = Wg[:, 1]          # duplicated columns tie exactly: lower id must win
    Wg[:, 5] = Wg[:, 0]
    X[0] = 0.0                   # all-zero token: every logit ties
    L = moe.gate_logits(X, Wg)
    assert np.array_equal(moe.top_k(L, k), _topk_by_rank_count(L, k))
    assert list(moe.top_k(L, k)[0]) == list(range(k))


def test_gate_weights_closed_forms():
    rng = np.random.default_rng(3)
    T, d, E = 50, 32, 8
    X = rng.standard_normal((T, d))
    X[0] = 0.0
    Wg = rng.standard_normal((d, E)) / math.sqrt(d)
    L = moe.gate_logits(X, Wg)
    p = moe.softmax(L)
    # k = 1: raw probability of the argmax (Switch)
    idx1 = moe.top_k(L, 1)
    g1 = moe.gate_weights(p, idx1)
    assert np.allclose(g1[:, 0], p.max(axis=1), rtol=1e-7)
    assert g1[0, 0] == pytest.approx(1.0 / E, rel=1e-6)
    # k = 2: weights sum to 1 and their ratio is exp(L0 − L1)  (softmax ratio, Z cancels)
    idx2 = moe.top_k(L, 2)
    g2 = moe.gate_weights(p, idx2)
    assert np.allclose(g2.sum(1), 1.0, atol=1e-6)
    l0 = np.take_along_axis(L, idx2[:, :1].astype(np.int64), 1)[:, 0]
    l1 = np.take_along_axis(L, idx2[:, 1:].astype(np.int64), 1)[:, 0]
    assert np.allclose(g2[:, 0] / g2[:, 1], np.exp(l0 - l1), rtol=1e-5)
    assert np.allclose(g2[0], [0.5, 0.5], atol=1e-7)


# ---------------------------------------------------------------- capacity


def test_capacity_golden(golden_dir):
    case = json.load(open(os.path.join(golden_dir, "capacity_case1.json")))
    slot, counts = moe.capacity_slots(np.array(case["idx"]), case["E"], case["C"])
    assert slot.tolist() == case["slot"]
    assert counts.tolist() == case["counts"]


@pytest.mark.parametrize("seed", range(20))
def test_capacity_brute_force_invariants(seed):
    rng = np.random.default_rng(100 + seed)
    T = int(rng.integers(1, 17)); E = int(rng.integers(1, 5)); k = int(rng.integers(1, min(E, 2) + 1))
    C = int(rng.integers(1, T + 2))
    idx = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    slot, counts = moe.capacity_slots(idx, E, C)
    # priority order enumerated independently: sort assignments by (j, t)
    order = sorted(((j, t) for t in range(T) for j in range(k)))
    assert counts.tolist() == [int((idx == e).sum()) for e in range(E)]
    for e in range(E):
        seq = [(t, j) for (j, t) in order if idx[t, j] == e]
        for n, (t, j) in enumerate(seq):             # kept set = prefix of the priority order
            assert slot[t, j] == (n if n < C else -1)
        kept = sorted(slot[t, j] for (t, j) in seq if slot[t, j] >= 0)
        assert kept == list(range(min(len(seq), C)))
    if C >= T:
        assert (slot >= 0).all()


# ---------------------------------------------------------------- layer special cases


def _identity_experts(E, d, f):
    W1 = np.zeros((E, f, d)); W2 = np.zeros((E, d, f))
    for e in range(E):
        W1[e, :d] = np.eye(d); W1[e, d:2 * d] = -np.eye(d)
        W2[e, :, :d] = np.eye(d); W2[e, :, d:2 * d] = -np.eye(d)
    return W1, W2


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_identity_experts_roundtrip(dtype):
    """P5: relu(x) − relu(−x) = x, so y_t = x_t · Σ_kept g (north_star invariant)."""
    cfg = li.with_tokens(li.CONFIGS["C1"], 96, k=2, num_experts=4, dtype=dtype)
    X, _ = li.layer_tokens(cfg, 7, 0)
    Wg, _, _ = li.layer_weights(cfg, 7)
    W1, W2 = _identity_experts(4, cfg.d_model, cfg.d_ffn)
    C = cfg.capacity()
    fw = moe.moe_forward([X], Wg, W1, W2, 2, C, dtype)[0]
    assert (fw.slot < 0).any() and (fw.slot >= 0).any()      # both kept and dropped rows
    gsum = (fw.gate * (fw.slot >= 0)).sum(1, keepdims=True)
    ref = X.astype(np.float64) * gsum
    ulp = 2.0 ** -8 if dtype == "bf16" else 2.0 ** -23
    assert np.all(np.abs(fw.y - ref) <= ulp * np.abs(ref) + 1e-30)


def test_dense_special_case_matches_textbook_ffn():
    """P6: E=1, k=1, C>=T  =>  p=1, g=1, y = relu(x W1ᵀ) W2ᵀ (torch fp64 as the textbook FFN)."""
    rng = np.random.default_rng(4)
    T, d, f = 33, 16, 48
    X = rng.standard_normal((T, d)); Wg = rng.standard_normal((d, 1))
    W1 = rng.standard_normal((1, f, d)); W2 = rng.standard_normal((1, d, f))
    fw = moe.moe_forward([X], Wg, W1, W2, 1, T, "f64")[0]
    ref = torch.nn.functional.linear(torch.relu(torch.nn.functional.linear(
        torch.from_numpy(X), torch.from_numpy(W1[0]))), torch.from_numpy(W2[0])).numpy()
    assert np.allclose(fw.gate, 1.0)
    assert np.allclose(fw.y, ref, rtol=1e-12, atol=1e-12)


def test_identical_experts_k2_equals_ffn():
    """P7: all experts equal, k=2, no drops  =>  Σg = 1  =>  y = FFN(x)."""
    rng = np.random.default_rng(5)
    T, d, f, E = 30, 8, 24, 4
    X = rng.standard_normal((T, d)); Wg = rng.standard_normal((d, E))
    w1 = rng.standard_normal((f, d)); w2 = rng.standard_normal((d, f))
    W1 = np.stack([w1] * E); W2 = np.stack([w2] * E)
    fw = moe.moe_forward([X], Wg, W1, W2, 2, T, "f64")[0]
    ref = np.maximum(X @ w1.T, 0) @ w2.T
    assert np.allclose(fw.y, ref, rtol=1e-6, atol=1e-6)   # g is fp32 (R2): Σg = 1 ± 1e-7


def test_multi_rank_capacity_is_per_source_rank():
    """Capacity counts are per source rank (each rank dispatches its own tokens):
    a two-rank run equals two independent one-rank runs row for row."""
    cfg = li.with_tokens(li.CONFIGS["C1"], 64)
    Wg, W1, W2 = li.layer_weights(cfg, 9)
    Xs = [li.layer_tokens(cfg, 9, r)[0] for r in range(2)]
    C = cfg.capacity()
    both = moe.moe_forward(Xs, Wg, W1, W2, 1, C, "f32")
    for r in range(2):
        one = moe.moe_forward([Xs[r]], Wg, W1, W2, 1, C, "f32")[0]
        assert np.array_equal(one.slot, both[r].slot)
        assert np.array_equal(one.y, both[r].y)


# ---------------------------------------------------------------- backward


def _loss(Xs, Wg, W1, W2, k, C, dYs):
    outs = moe.moe_forward(Xs, Wg, W1, W2, k, C, "f64")
    return sum(float((o.y * dY).sum()) for o, dY in zip(outs, dYs)), outs


@pytest.mark.parametrize("k", [1, 2])
def test_backward_central_finite_differences(k):
    """P10: fp64 central differences of <y, dY> w.r.t. X, Wg, W1, W2 (2 ranks, with drops)."""
    rng = np.random.default_rng(10 + k)
    T, d, f, E, P = 12, 6, 10, 4, 2
    C = 4 if k == 2 else 3
    Xs = [rng.standard_normal((T, d)) for _ in range(P)]
    dYs = [rng.standard_normal((T, d)) for _ in range(P)]
    Wg = rng.standard_normal((d, E)); W1 = rng.standard_normal((E, f, d)); W2 = rng.standard_normal((E, d, f))
    _, outs = _loss(Xs, Wg, W1, W2, k, C, dYs)
    assert any((o.slot < 0).any() for o in outs)
    bw = moe.moe_backward(outs, Xs, dYs, Wg, W1, W2, k, "f64")
    eps = 1e-6

    def fd(arr, i, setter):
        old = arr[i]
        arr[i] = old + eps; setter(); lp, op = _loss(Xs, Wg, W1, W2, k, C, dYs)
        arr[i] = old - eps; setter(); lm, om = _loss(Xs, Wg, W1, W2, k, C, dYs)
        arr[i] = old
        for a, b, c in zip(op, om, outs):              # routing must not move within ±eps
            assert np.array_equal(a.idx, c.idx) and np.array_equal(b.idx, c.idx)
        return (lp - lm) / (2 * eps)

    nop = lambda: None
    for (r, t, c) in [(0, 0, 0), (1, 5, 3), (0, 11, 5), (1, 2, 1)]:
        assert fd(Xs[r], (t, c), nop) == pytest.approx(bw.dXs[r][t, c], rel=1e-5, abs=1e-7)
    for i in [(0, 0), (3, 2), (5, 3), (2, 1)]:
        assert fd(Wg, i, nop) == pytest.approx(bw.dWg[i], rel=1e-5, abs=1e-6)
    for i in [(0, 0, 0), (1, 3, 2), (2, 9, 5), (3, 4, 4)]:
        assert fd(W1, i, nop) == pytest.approx(bw.dW1[i], rel=1e-5, abs=1e-7)
    for i in [(0, 0, 0), (1, 2, 7), (2, 5, 9), (3, 1, 3)]:
        assert fd(W2, i, nop) == pytest.approx(bw.dW2[i], rel=1e-5, abs=1e-7)


def test_backward_gate_closed_form_k2():
    """Q13 closed form for k>=2: dL_{e_j} = g_j (dg_j − Σ g dg), dL = 0 off the selected set.
    Checked through dWg = Xᵀ dL on a one-token batch."""
    rng = np.random.default_rng(21)
    d, f, E = 5, 7, 4
    X = rng.standard_normal((1, d)); dY = rng.standard_normal((1, d))
    Wg = rng.standard_normal((d, E)); W1 = rng.standard_normal((E, f, d)); W2 = rng.standard_normal((E, d, f))
    outs = moe.moe_forward([X], Wg, W1, W2, 2, 1, "f64")
    bw = moe.moe_backward(outs, [X], [dY], Wg, W1, W2, 2, "f64")
    o = outs[0]; g = o.gate[0]; dg = bw.dgs[0][0]
    dL = np.zeros(E)
    for j in range(2):
        dL[o.idx[0, j]] = g[j] * (dg[j] - (g * dg).sum())
    assert np.allclose(bw.dWg, X.T @ dL[None, :], rtol=1e-6, atol=1e-9)


# ---------------------------------------------------------------- placement


def test_placement_golden(golden_dir):
    cases = json.load(open(os.path.join(golden_dir, "placement_cases.json")))["cases"]
    for c in cases:
        plan = placement.place(c["popularity"], c["N"], c["max_per_device"])
        assert plan["replicas"] == c["replicas"]
        assert plan["hosted"] == c["hosted"]


def test_placement_infeasible():
    with pytest.raises(placement.InfeasiblePlan):
        placement.place([0.1] * 10, 2, 4)


@pytest.mark.parametrize("seed", range(30))
def test_placement_invariants(seed):
    rng = np.random.default_rng(300 + seed)
    N = int(rng.integers(1, 9)); mpd = int(rng.integers(1, 5))
    E = int(rng.integers(1, N * mpd + 1))
    pop = rng.dirichlet(np.full(E, 0.3))
    pop[rng.random(E) < 0.2] = 0.0
    pop = pop / pop.sum() if pop.sum() > 0 else np.full(E, 1.0 / E)
    plan = placement.place(list(pop), N, mpd)
    assert all(r >= 1 for r in plan["replicas"])
    assert all(len(h) <= mpd and len(set(h)) == len(h) for h in plan["hosted"])
    for e in range(E):
        assert len(plan["replica_device"][e]) == plan["replicas"][e]
    # token split: sizes differ by <= 1 and sum to the count
    for s in range(3):
        for e in range(E):
            cnt = int(rng.integers(0, 50))
            sp = placement.replica_split(cnt, plan["replicas"][e], s)
            assert sum(sp) == cnt and max(sp) - min(sp) <= 1


def _opt_bins(sizes):
    """Brute-force minimum number of unit bins (tiny instances)."""
    n = len(sizes)
    for b in range(1, n + 1):
        for assign in itertools.product(range(b), repeat=n):
            loads = [0.0] * b
            for s, a in zip(sizes, assign):
                loads[a] += s
            if max(loads) <= 1.0 + 1e-9:
                return b
    return n


@pytest.mark.parametrize("seed", range(25))
def test_ffd_within_known_bound_of_brute_force_optimum(seed):
    """FFD(I) <= 11/9 OPT(I) + 6/9 (Dósa 2007) on unit bins, replicas all 1 (no trimming),
    enough devices and slots that first fit never overflows."""
    rng = np.random.default_rng(500 + seed)
    E = int(rng.integers(1, 7)); N = 8
    # sizes n_e = N·pop_e in (0, 1): round-half-up gives r_e = 1 when n_e < 0.5 only, so keep them small
    sizes = rng.uniform(0.05, 0.49, size=E)
    pop = sizes / N
    plan = placement.place(list(pop), N, E)
    used = sum(1 for h in plan["hosted"] if h)
    assert used <= 11 / 9 * _opt_bins(list(sizes)) + 6 / 9 + 1e-9


# ---------------------------------------------------------------------------
# Pins of the comparison metric and of the replica token split (unpinned)
# ---------------------------------------------------------------------------


def test_normwise_error_hand_cases():
    """north_star's metric (SURVEY.md §8(c) "Tolerances"): max_i |got_i − ref_i| / max_i |ref_i|.
    The cases are chosen so a mean for a max, |got| in the denominator or an element-wise
    relative error each give a different value."""
    assert moe.normwise_error([1.0, 2.0, 3.0], [1.0, 2.0, 4.0]) == 0.25
    # diffs (1, 1, 10), max|ref| = 20: 0.5 (mean of diffs 4/20 = 0.2; max|got| denominator
    # 10/10 = 1; element-wise max |d|/|r| = 1)
    assert moe.normwise_error([0.0, 0.0, 10.0], [1.0, 1.0, 20.0]) == 0.5
    assert moe.normwise_error([0.0, -3.0], [1.0, -2.0]) == 0.5           # signs: |−3 − (−2)| = 1
    assert moe.normwise_error(np.array([[1.0, 5.0], [2.0, 2.0]]), np.array([[1.0, 4.0], [2.0, 8.0]])) == 0.75
    assert moe.normwise_error([0.5, 0.0], [0.0, 0.0]) == 0.5             # zero reference: absolute
    assert moe.normwise_error([], []) == 0.0


@pytest.mark.parametrize("count,r,s,expect", [
    (7, 3, 0, [3, 2, 2]),      # blocks (3, 2, 2) in slot order, block q -> replica q
    (7, 3, 1, [2, 3, 2]),      # block q -> replica (q + 1) mod 3
    (7, 3, 2, [2, 2, 3]),
    (7, 3, 4, [2, 3, 2]),      # s = 4 rotates like s = 1
    (5, 2, 1, [2, 3]),
    (1, 4, 3, [0, 0, 0, 1]),
    (0, 3, 1, [0, 0, 0]),
    (8, 4, 2, [2, 2, 2, 2]),
])
def test_replica_split_rotation_hand_table(count, r, s, expect):
    """R14 ("how many tokens each replica should handle to balance the load"):
    contiguous blocks differing by <= 1, block q to replica (q + s) mod r_e."""
    assert placement.replica_split(count, r, s) == expect


def test_replica_split_rotation_balances_remainders_across_sources():
    """With one token per source and r_e sources, the rotation gives every replica exactly one
    token; any split without the rotation puts all of them on replica 0."""
    for r in (2, 3, 5):
        tot = np.zeros(r, int)
        for s in range(r):
            tot += placement.replica_split(1, r, s)
        assert tot.tolist() == [1] * r


def test_route_counts_hand_case():
    """send[s][dv][e] for two sources, expert 0 replicated on devices {0, 1}, expert 1 on {1}."""
    plan = {"replicas": [2, 1], "replica_device": [[0, 1], [1]]}
    send = placement.route_counts([[5, 3], [4, 2]], plan, 2)
    # source 0: e0 5 tokens -> blocks (3, 2) to replicas (0, 1); e1 -> device 1
    # source 1: e0 4 tokens -> blocks (2, 2) to replicas (1, 0); e1 -> device 1
    assert send == [[[3, 0], [2, 3]], [[2, 0], [2, 2]]]
