"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the MoE method (no gating, routing, FFN,
combine or placement).  It only draws random tensors with the shapes and value
distributions of the paper's workloads and holds the
config table from BASELINE.json.  Both ``oracle/`` and the CUDA path receive
the same arrays from here; neither imports the other.

Families
--------
grid      : every value on {k/64 : |k| <= 31} (expert weights additionally /8).
            Exact in bf16, and every fp32 gate logit is exact under any
            summation order, so routing parity is bit-exact.
balanced  : X ~ N(0,1), Wg ~ N(0,1/d), W1 ~ N(0,1/d), W2 ~ N(0,1/f): near-uniform
            routing, as in training ("nearly the same across all experts",
            PAPER.md:243 §2.2).
zipf      : z_t ~ Zipf(s) over experts, X_t = 6 u_{z_t} + N(0, I), Wg[:, e] = u_e.
            Reproduces the skewed inference popularity of PAPER.md:243 (§2.2).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# ----------------------------------------------------------------------------
# Config table (BASELINE.json "configs"; SURVEY.md §8 glossary).  Values marked
# "proposed" in SURVEY.md §8 are the readings recorded in DESIGN.md.
# ----------------------------------------------------------------------------


@dataclass(frozen=True)
class LayerConfig:
    name: str
    num_experts: int      # E (global)
    k: int                # top-k
    d_model: int          # d
    d_ffn: int            # f
    tokens_per_rank: int  # T
    cf: float | None      # capacity factor; None => dropless (C = T)
    dtype: str            # "f32" | "bf16"

    def capacity(self) -> int:
        """C = ceil(cf * k * T / E) slots per expert per source rank (R5)."""
        if self.cf is None:
            return self.tokens_per_rank
        return int(math.ceil(self.cf * self.k * self.tokens_per_rank / self.num_experts))


CONFIGS = {
    # configs[0]: tiny, fp32, CPU oracle in seconds.  cf=1.0 gives drops.
    "C1": LayerConfig("C1-tiny", 4, 1, 64, 256, 512, 1.0, "f32"),
    # configs[1]: GPT-2-small-shaped, 8 experts (1/GPU at 8 GPUs), top-2, d=768, 8K tok/GPU, bf16.
    "C2": LayerConfig("C2-gpt2s", 8, 2, 768, 3072, 8192, 1.25, "bf16"),
    # configs[2]: BERT-large-shaped, 16 experts, top-2, d=1024, capacity 1.25.
    "C3": LayerConfig("C3-bertl", 16, 2, 1024, 4096, 8192, 1.25, "bf16"),
    # configs[3]: Transformer-XL-shaped inference, 32 experts, top-1, dropless.
    "C4": LayerConfig("C4-txl-inf", 32, 1, 1024, 4096, 4096, None, "bf16"),
    # configs[4]: scale sweep.
    "C5": LayerConfig("C5-scale", 64, 2, 2048, 8192, 32768, 1.25, "bf16"),
}


# ----------------------------------------------------------------------------
# Random draws
# ----------------------------------------------------------------------------


def _rng(seed: int, *stream: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([int(seed), *[int(s) for s in stream]]))


def bf16_representable(a: np.ndarray) -> np.ndarray:
    """Round float32 data to the nearest bf16 value (RNE), returned as float32.

    Data preparation only: makes a random draw storable in bf16 without loss, so
    both sides start from identical values.
    """
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def grid(rng: np.random.Generator, shape, scale: float = 1.0) -> np.ndarray:
    """Uniform on {k/64 : |k| <= 31} * scale (scale a power of two keeps bf16 exactness)."""
    k = rng.integers(-31, 32, size=shape, dtype=np.int64)
    return (k.astype(np.float64) / 64.0 * scale).astype(np.float32)


TENSOR_IDS = {"X": 1, "Wg": 2, "W1": 3, "W2": 4, "dY": 5, "zipf": 6, "trace": 7}


def gate_weight(cfg: LayerConfig, seed: int, family: str = "grid") -> np.ndarray:
    """Wg [d,E] fp32, identical on every rank."""
    d, E = cfg.d_model, cfg.num_experts
    if family == "grid":
        return grid(_rng(seed, TENSOR_IDS["Wg"]), (d, E))
    if family == "balanced":
        return (_rng(seed, TENSOR_IDS["Wg"]).standard_normal((d, E)) / math.sqrt(d)).astype(np.float32)
    if family == "zipf":
        return np.ascontiguousarray(_zipf_directions(cfg, seed).T).astype(np.float32)
    raise ValueError(f"unknown family {family!r}")


def expert_weights(cfg: LayerConfig, seed: int, e: int, family: str = "grid"):
    """Expert e's W1 [f,d] and W2 [d,f] (each expert drawn from its own stream, so a rank
    can generate just the experts it hosts)."""
    d, f = cfg.d_model, cfg.d_ffn
    r1, r2 = _rng(seed, TENSOR_IDS["W1"], e), _rng(seed, TENSOR_IDS["W2"], e)
    if family == "grid":
        W1 = grid(r1, (f, d), 1.0 / 8)
        W2 = grid(r2, (d, f), 1.0 / 8)
    elif family in ("balanced", "zipf"):
        W1 = r1.standard_normal((f, d), dtype=np.float32) / np.float32(math.sqrt(d))
        W2 = r2.standard_normal((d, f), dtype=np.float32) / np.float32(math.sqrt(f))
    else:
        raise ValueError(f"unknown family {family!r}")
    if cfg.dtype == "bf16":
        W1 = bf16_representable(W1)
        W2 = bf16_representable(W2)
    return W1, W2


def layer_weights(cfg: LayerConfig, seed: int, family: str = "grid", experts=None):
    """Wg [d,E] fp32 and the stacked W1 [n,f,d], W2 [n,d,f] of `experts` (default: all E)."""
    experts = range(cfg.num_experts) if experts is None else experts
    ws = [expert_weights(cfg, seed, e, family) for e in experts]
    W1 = np.stack([w[0] for w in ws])
    W2 = np.stack([w[1] for w in ws])
    return gate_weight(cfg, seed, family), W1, W2


def _zipf_directions(cfg: LayerConfig, seed: int) -> np.ndarray:
    U = _rng(seed, TENSOR_IDS["zipf"], 0).standard_normal((cfg.num_experts, cfg.d_model))
    U /= np.linalg.norm(U, axis=1, keepdims=True)
    return U


def zipf_probs(E: int, s: float) -> np.ndarray:
    w = 1.0 / np.arange(1, E + 1, dtype=np.float64) ** s
    return w / w.sum()


def layer_tokens(cfg: LayerConfig, seed: int, rank: int, family: str = "grid",
                 zipf_s: float = 1.0, num_tokens: int | None = None):
    """Per-rank tokens X [T,d] and upstream gradient dY [T,d] (bf16-representable when dtype=bf16)."""
    T = cfg.tokens_per_rank if num_tokens is None else num_tokens
    d = cfg.d_model
    if family == "grid":
        X = grid(_rng(seed, TENSOR_IDS["X"], rank), (T, d))
        dY = grid(_rng(seed, TENSOR_IDS["dY"], rank), (T, d))
    elif family == "balanced":
        X = _rng(seed, TENSOR_IDS["X"], rank).standard_normal((T, d), dtype=np.float32)
        dY = _rng(seed, TENSOR_IDS["dY"], rank).standard_normal((T, d), dtype=np.float32)
    elif family == "zipf":
        rng = _rng(seed, TENSOR_IDS["X"], rank)
        U = _zipf_directions(cfg, seed)
        z = rng.choice(cfg.num_experts, size=T, p=zipf_probs(cfg.num_experts, zipf_s))
        X = (6.0 * U[z] + rng.standard_normal((T, d))).astype(np.float32)
        dY = _rng(seed, TENSOR_IDS["dY"], rank).standard_normal((T, d), dtype=np.float32)
    else:
        raise ValueError(f"unknown family {family!r}")
    if cfg.dtype == "bf16":
        X = bf16_representable(X)
        dY = bf16_representable(dY)
    return X, dY


def with_tokens(cfg: LayerConfig, tokens: int, **changes) -> LayerConfig:
    """A reduced copy of a config (parity cases at sizes the oracle finishes in seconds)."""
    fields = dict(cfg.__dict__)
    fields["tokens_per_rank"] = tokens
    fields.update(changes)
    return LayerConfig(**fields)


# ----------------------------------------------------------------------------
# Expert-selection traces (inputs of the popularity profiler / estimator, §8(f) row 2)
# ----------------------------------------------------------------------------


@dataclass
class SelectionTrace:
    """sel[t][i] = the k experts token t selected in MoE layer i (int32 [T, L, k]).

    Generated by a first-order Markov model (SPEC.md's generator idea): each layer i >= 1
    has a fixed random map ``maps[i-1]`` from the token's previous first expert to a
    follow-on expert; with probability ``p`` the token's first expert follows the map,
    else it is drawn from the layer's Zipf(zipf_s) marginal ``marginal`` (expert ids
    permuted per layer).  The remaining k-1 experts are drawn from the same marginal
    without replacement.  Layer 0 draws from its marginal.  The maps and marginals are
    returned so tests can state the ground-truth next-layer distribution in closed form.
    """
    sel: np.ndarray
    maps: np.ndarray       # [L-1, E] follow-on expert of layer i+1 given first expert a in layer i
    marginal: np.ndarray   # [L, E]   Zipf marginal of each layer (permuted expert ids)
    p: float


def selection_trace(num_tokens: int, num_layers: int, num_experts: int, k: int, p: float,
                    zipf_s: float, seed: int, stream: int = 0, maps=None, marginal=None) -> SelectionTrace:
    """Seeded trace; pass ``maps``/``marginal`` of another trace to draw a fresh batch from
    the same model (a profiling trace and an inference batch share the model)."""
    T, L, E = num_tokens, num_layers, num_experts
    if not (0.0 <= p <= 1.0) or not (1 <= k <= E):
        raise ValueError("need 0 <= p <= 1 and 1 <= k <= E")
    mrng = _rng(seed, TENSOR_IDS["trace"], 0)
    if maps is None:
        maps = np.stack([mrng.integers(0, E, size=E) for _ in range(max(L - 1, 0))]) \
            if L > 1 else np.zeros((0, E), dtype=np.int64)
    if marginal is None:
        z = zipf_probs(E, zipf_s)
        marginal = np.stack([z[np.argsort(mrng.permutation(E))] for _ in range(L)])
    rng = _rng(seed, TENSOR_IDS["trace"], 1 + stream)
    sel = np.empty((T, L, k), dtype=np.int32)
    for i in range(L):
        first = rng.choice(E, size=T, p=marginal[i])
        if i > 0 and p > 0:
            follow = rng.random(T) < p
            first = np.where(follow, maps[i - 1][sel[:, i - 1, 0]], first)
        sel[:, i, 0] = first
        for t in range(T) if k > 1 else ():
            w = marginal[i].copy()
            w[first[t]] = 0.0
            sel[t, i, 1:] = rng.choice(E, size=k - 1, replace=False, p=w / w.sum())
    return SelectionTrace(sel, np.asarray(maps), np.asarray(marginal), p)
