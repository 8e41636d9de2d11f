"""Host logic of bench.py (no GPU): the roofline floors of the expert-GEMM family.

The byte count is pinned by brute force — summing the operand and result tensors of the
six GEMMs written out one by one — not by retyping the closed form.
"""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PK = {"bf16_sustained": 1408.6, "bf16_burst": 1683.0, "hbm": 6459.3, "src": "test"}


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_under_test", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _gemm_tensors(d, f, el, rows, elt):
    """Bytes each GEMM reads and writes, listed per tensor (shape products × element size)."""
    W = el * d * f * elt          # one of W1 [El,f,d], W2 [El,d,f], dW1, dW2
    x, h = rows * d * elt, rows * f * elt
    mask = rows * f / 8
    return [
        ("GEMM1  H = relu(X W1^T)", [x, W], [h, mask]),
        ("GEMM2  Y = H W2^T", [h, W], [x]),
        ("dgrad1 dH = (dY W2) * relu'", [x, W, mask], [h]),
        ("dgrad2 dX = dH W1", [h, W], [x]),
        ("wgrad1 dW1 = dH^T X", [h, x], [W]),
        ("wgrad2 dW2 = dY^T H", [x, h], [W]),
    ]


@pytest.mark.parametrize("d,f,el,rows", [(768, 3072, 8, 16384), (1024, 4096, 32, 4096), (64, 256, 4, 512)])
def test_gemm_bytes_brute_force(bench, d, f, el, rows):
    fl = bench.gemm_floors(d, f, el, rows, 2, PK, PK["bf16_sustained"])
    brute = sum(sum(i) + sum(o) for _, i, o in _gemm_tensors(d, f, el, rows, 2))
    assert fl["bytes"] == pytest.approx(brute, rel=1e-12)
    assert fl["flops"] == 6 * (2.0 * rows * d * f)      # six GEMMs of 2·rows·d·f flop each


def test_bound_selection(bench):
    c2 = bench.gemm_floors(768, 3072, 8, 16384, 2, PK, PK["bf16_sustained"])     # C2, N=1: long segments
    assert not c2["hbm_bound"] and c2["tensor_ms"] == pytest.approx(0.3293, rel=1e-3)
    c4 = bench.gemm_floors(1024, 4096, 32, 4096, 2, PK, PK["bf16_sustained"])    # C4 as a layer: ~128 rows per expert
    assert c4["hbm_bound"] and c4["hbm_ms"] > 1.9 * c4["tensor_ms"]
    # crossover: the ridge point of the pair of peaks (flop per byte) decides
    ridge = PK["bf16_sustained"] * 1e12 / (PK["hbm"] * 1e9)
    for rows in (512, 2048, 8192, 65536):
        fl = bench.gemm_floors(1024, 4096, 32, rows, 2, PK, PK["bf16_sustained"])
        assert fl["hbm_bound"] == (fl["flops"] / fl["bytes"] < ridge)


def test_peak_choice_follows_the_clock_record(bench):
    pk = dict(PK)
    burst = bench.choose_peak(pk, {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0, "reasons": []})
    assert burst[:2] == (PK["bf16_burst"], "burst")
    capped = bench.choose_peak(pk, {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0, "reasons": ["sw_power_cap"]})
    assert capped[:2] == (PK["bf16_sustained"], "sustained")
    slow = bench.choose_peak(pk, {"sm_mhz": 1327.0, "sm_max_mhz": 1965.0, "reasons": []})
    assert slow[:2] == (PK["bf16_sustained"], "sustained")


def test_layer_floor_terms_brute_force(bench):
    """§8(d) layer roofline: each term from the kernels' tensors listed one by one."""
    d, f, El, k, T, P, elt = 2048, 8192, 8, 2, 32768, 8, 2
    kept = T * k - 1000                           # some drops
    lf = bench.layer_floor(d, f, El, k, T, kept, P, elt, 1000.0, 5000.0)
    row = d * elt
    fwd = [T * row,                               # gate reads X
           T * row, k * T * row,                  # permute reads X, writes k rows per token
           k * T * row, T * row]                  # combine reads k rows, writes y
    bwd = [T * row, k * T * row, k * T * row,     # combine-backward: dY, k outputs in, k rows out
           k * T * row, T * row,                  # dX: k rows in, dX out
           T * row]                               # dWg reads X
    assert lf["memkernel_bytes"] == sum(fwd) + sum(bwd)
    assert lf["a2a_bytes_per_direction"] == pytest.approx(4 * kept * row * (P - 1) / P)
    assert lf["gemm_flops"] == 12.0 * kept * d * f
    t = max(lf["gemm_flops"] / 1e15, lf["a2a_bytes_per_direction"] / 900e9) + (sum(fwd) + sum(bwd)) / 5e12
    assert lf["t_roof_ms"] == pytest.approx(t * 1e3, rel=1e-12)
    # P = 1: no off-GPU bytes
    assert bench.layer_floor(d, f, El, k, T, kept, 1, elt, 1000.0, 5000.0)["a2a_bytes_per_direction"] == 0
