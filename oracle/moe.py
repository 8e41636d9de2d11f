"""Oracle MoE layer (forward + backward) — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Written step by step from PAPER.md §2.1 and §2.2's
"Gate ... reshaping the tensors and computing the weighted output",
with the readings R1-R13 listed in DESIGN.md §3 where the paper is silent.

All P source ranks are simulated in one process: routing and capacity are per
source rank (each rank gates its own tokens), experts are global.
The placement of experts on devices does not change any value (PAPER.md:646:
Lina "does not affect the precision of model parameters"), so this oracle has
no notion of chunks, streams, all-to-all or replicas.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# Rounding to the storage dtype (R8)
# ---------------------------------------------------------------------------


def round_bf16(x) -> np.ndarray:
    """Round fp64 values to the nearest bf16 (8 significant bits), ties to even."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)                       # x = m * 2**e, 0.5 <= |m| < 1
    m = np.rint(m * 256.0) / 256.0           # keep 8 significant bits, RNE
    return np.ldexp(m, e)


def round_to(x, dtype: str) -> np.ndarray:
    """dtype in {"f64", "f32", "bf16"}; returns fp64 arrays holding the rounded values."""
    x = np.asarray(x, dtype=np.float64)
    if dtype == "f64":
        return x
    if dtype == "f32":
        return x.astype(np.float32).astype(np.float64)
    if dtype == "bf16":
        return round_bf16(x)
    raise ValueError(dtype)


# ---------------------------------------------------------------------------
# Step 1-4: gating network (§2.1)
# ---------------------------------------------------------------------------


def gate_logits(X, Wg, prec: str = "f32") -> np.ndarray:
    """L = X · Wg  ("multiplies them with its trainable matrix").

    No bias, no noise (R1).  fp64 accumulation, rounded to fp32 (R2: the gate is
    fp32 on every path)."""
    return round_to(np.asarray(X, np.float64) @ np.asarray(Wg, np.float64), prec)


def softmax(L, prec: str = "f32") -> np.ndarray:
    """p = softmax(L) over all E experts with max-subtraction (R1), fp64, rounded to fp32."""
    L = np.asarray(L, np.float64)
    z = np.exp(L - L.max(axis=1, keepdims=True))
    return round_to(z / z.sum(axis=1, keepdims=True), prec)


def top_k(L, k: int) -> np.ndarray:
    """Select k experts per token ("dispatches the token to a small number of experts").

    Order: logit descending, expert id ascending on ties (R3).  Keyed on the
    logits, never on the probabilities."""
    L = np.asarray(L, np.float64)
    T, E = L.shape
    idx = np.empty((T, k), dtype=np.int32)
    for t in range(T):
        order = sorted(range(E), key=lambda e: (-L[t, e], e))
        idx[t] = order[:k]
    return idx


def gate_weights(p, idx, prec: str = "f32") -> np.ndarray:
    """Weights of the selected experts ("weighted sum of outputs from the selected expert(s)").

    k=1: g = p[e0] (Switch, cited for k=1 at P:556).  k>=2: renormalised over
    the k selected experts, before any capacity drop (R4).  Rounded to fp32."""
    p = np.asarray(p, np.float64)
    T, k = idx.shape
    sel = np.take_along_axis(p, idx.astype(np.int64), axis=1)
    if k == 1:
        g = sel
    else:
        g = sel / sel.sum(axis=1, keepdims=True)
    return round_to(g, prec)


# ---------------------------------------------------------------------------
# Step 5: capacity-bounded slot assignment (R5, R6)
# ---------------------------------------------------------------------------


def capacity_slots(idx, num_experts: int, capacity: int):
    """Per source rank: for j = 0..k-1, then t = 0..T-1: slot = cnt[e]++; kept iff slot < C.

    Returns slot[T,k] (int32, -1 = dropped) and counts[E] (pre-drop totals)."""
    T, k = idx.shape
    cnt = [0] * num_experts
    slot = np.full((T, k), -1, dtype=np.int32)
    for j in range(k):
        for t in range(T):
            e = int(idx[t, j])
            s = cnt[e]
            cnt[e] += 1
            if s < capacity:
                slot[t, j] = s
    return slot, np.asarray(cnt, dtype=np.int32)


# ---------------------------------------------------------------------------
# Step 7: experts — "a fully-connected two-layer network using ReLU"
# ---------------------------------------------------------------------------


def expert_ffn(x_rows, W1e, W2e, dtype: str):
    """h = relu(x · W1eᵀ) (rounded to dtype), o = h · W2eᵀ (rounded to dtype).  No biases (R8)."""
    h = round_to(np.maximum(np.asarray(x_rows, np.float64) @ np.asarray(W1e, np.float64).T, 0.0), dtype)
    o = round_to(h @ np.asarray(W2e, np.float64).T, dtype)
    return h, o


# ---------------------------------------------------------------------------
# Forward of the whole layer over P source ranks
# ---------------------------------------------------------------------------


@dataclass
class RankForward:
    L: np.ndarray       # [T,E] fp32 logits
    p: np.ndarray       # [T,E] fp32 probabilities
    idx: np.ndarray     # [T,k] int32
    gate: np.ndarray    # [T,k] fp32
    slot: np.ndarray    # [T,k] int32, -1 = dropped
    counts: np.ndarray  # [E] int32 pre-drop
    y: np.ndarray       # [T,d] output (values of dtype)
    h: dict = field(default_factory=dict)   # (t,j) -> h row   (kept only)
    o: dict = field(default_factory=dict)   # (t,j) -> o row   (kept only)


def moe_forward(Xs, Wg, W1, W2, k: int, capacity: int, dtype: str):
    """MoE layer forward: gate -> top-k -> capacity -> experts -> weighted sum.

    Xs: list over source ranks of [T,d] token arrays.  W1 [E,f,d], W2 [E,d,f]
    hold all E experts.  Returns a list of RankForward."""
    E = int(np.asarray(Wg).shape[1])
    prec = "f64" if dtype == "f64" else "f32"      # "f64" = exact-arithmetic mode for finite differences
    outs = []
    for X in Xs:
        X = np.asarray(X, np.float64)
        L = gate_logits(X, Wg, prec)
        p = softmax(L, prec)
        idx = top_k(L, k)
        g = gate_weights(p, idx, prec)
        slot, counts = capacity_slots(idx, E, capacity)
        outs.append(RankForward(L=L, p=p, idx=idx, gate=g, slot=slot, counts=counts,
                                y=np.zeros_like(X)))
    # Experts: each kept (rank, t, j) row goes to expert idx[t,j] (the dispatch all-to-all).
    X64 = [np.asarray(X, np.float64) for X in Xs]   # (once: a row of a per-row copy pins the copy)
    for e in range(E):
        rows = [(r, t, j) for r, fw in enumerate(outs)
                for t, j in zip(*np.nonzero((fw.idx == e) & (fw.slot >= 0)))]
        if not rows:
            continue
        x = np.stack([X64[r][t] for r, t, _ in rows])
        h, o = expert_ffn(x, W1[e], W2[e], dtype)
        for n, (r, t, j) in enumerate(rows):
            outs[r].h[(int(t), int(j))] = h[n]
            outs[r].o[(int(t), int(j))] = o[n]
    for fw in outs:
        fw.y = combine(fw, k, dtype)
    return outs


def combine(fw: "RankForward", k: int, dtype: str) -> np.ndarray:
    """The return all-to-all + "computing the weighted output":
    y_t = sum over kept j, ascending, of g[t,j] * o[t,j]; fp64, one final rounding (R9).
    A token whose k assignments were all dropped gets y_t = 0 (R7)."""
    T, d = fw.y.shape
    acc = np.zeros((T, d))
    for t in range(T):
        for j in range(k):
            if fw.slot[t, j] >= 0:
                acc[t] += fw.gate[t, j] * fw.o[(t, j)]
    return round_to(acc, dtype)


# ---------------------------------------------------------------------------
# Backward (chain rule through the forward above; R12, R13)
# ---------------------------------------------------------------------------


@dataclass
class Backward:
    dXs: list            # per rank [T,d]
    dWg: np.ndarray      # [d,E] fp32, summed over ranks (the allreduced value, R12)
    dW1: np.ndarray      # [E,f,d]
    dW2: np.ndarray      # [E,d,f]
    dgs: list            # per rank [T,k] fp32 gradient w.r.t. gate weights


def moe_backward(fw_outs, Xs, dYs, Wg, W1, W2, k: int, dtype: str) -> Backward:
    E = int(np.asarray(Wg).shape[1])
    Wg = np.asarray(Wg, np.float64)
    W1 = np.asarray(W1, np.float64)
    W2 = np.asarray(W2, np.float64)
    dW1 = np.zeros_like(W1)
    dW2 = np.zeros_like(W2)
    dWg = np.zeros_like(Wg)
    dXs, dgs = [], []
    dXe = [dict() for _ in fw_outs]
    # (a) y_t = sum_j g_tj o_tj  =>  dg_tj = <dY_t, o_tj>,  dO_tj = g_tj dY_t (rounded: it is stored)
    dO = [dict() for _ in fw_outs]
    for r, fw in enumerate(fw_outs):
        dY = np.asarray(dYs[r], np.float64)
        dg = np.zeros((dY.shape[0], k))
        for (t, j), o in fw.o.items():
            dg[t, j] = dY[t] @ o
            dO[r][(t, j)] = round_to(fw.gate[t, j] * dY[t], dtype)
        dgs.append(round_to(dg, "f64" if dtype == "f64" else "f32"))
    # (c) experts: dH = (dO · W2e) ∘ 1[h > 0], dXe = dH · W1e, dW2e = Σ dOᵀ h, dW1e = Σ dHᵀ x
    X64 = [np.asarray(X, np.float64) for X in Xs]
    for e in range(E):
        keys = [(r, t, j) for r, fw in enumerate(fw_outs) for (t, j) in fw.o
                if fw.idx[t, j] == e]
        if not keys:
            continue
        do = np.stack([dO[r][(t, j)] for r, t, j in keys])
        h = np.stack([fw_outs[r].h[(t, j)] for r, t, j in keys])
        x = np.stack([X64[r][t] for r, t, _ in keys])
        dh = round_to((do @ W2[e]) * (h > 0), dtype)          # relu'(0) = 0 (R8)
        dxe = round_to(dh @ W1[e], dtype)
        dW2[e] += do.T @ h
        dW1[e] += dh.T @ x
        for n, (r, t, j) in enumerate(keys):
            dXe[r][(t, j)] = dxe[n]
    # (e)+(f) per rank: dX_t = Σ_kept dXe + gate path; dWg = Σ_ranks Xᵀ dL
    for r, fw in enumerate(fw_outs):
        X = np.asarray(Xs[r], np.float64)
        T = X.shape[0]
        dg = dgs[r]
        # dg -> dp through g (R4/R13): k=1 g_0 = p_e0;  k>=2 g_j = p_ej / S, S = Σ_j' p_ej'
        dp = np.zeros((T, E))
        for t in range(T):
            sel = [int(fw.idx[t, j]) for j in range(k)]
            if k == 1:
                dp[t, sel[0]] += dg[t, 0]
            else:
                S = sum(fw.p[t, e] for e in sel)
                for i, ei in enumerate(sel):
                    for j, ej in enumerate(sel):
                        dgj_dpi = (1.0 if i == j else 0.0) / S - fw.p[t, ej] / S ** 2
                        dp[t, ei] += dg[t, j] * dgj_dpi
        # softmax Jacobian: dL = p ∘ (dp − <p, dp>)
        p = fw.p
        dL = p * (dp - (p * dp).sum(axis=1, keepdims=True))
        dWg += X.T @ dL
        acc = dL @ Wg.T
        for (t, j), v in dXe[r].items():
            acc[t] += v
        dXs.append(round_to(acc, dtype))
    return Backward(dXs=dXs, dWg=round_to(dWg, "f64" if dtype == "f64" else "f32"), dW1=round_to(dW1, dtype),
                    dW2=round_to(dW2, dtype), dgs=dgs)


# ---------------------------------------------------------------------------
# Helpers for comparisons
# ---------------------------------------------------------------------------


def normwise_error(got, ref) -> float:
    """max_i |got_i − ref_i| / max_i |ref_i| (north_star tolerance metric)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.abs(ref).max() if ref.size else 0.0
    num = np.abs(got - ref).max() if ref.size else 0.0
    return float(num / den) if den > 0 else float(num)
