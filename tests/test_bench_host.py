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
    fl = bench.gemm_floors(d, f, el, rows, 2, PK)
    brute = sum(sum(i) + sum(o) for _, i, o in _gemm_tensors(d, f, el, rows, 2))
    assert fl["bytes"] == pytest.approx(brute, rel=1e-12)
    assert fl["flops"] == 6 * (2.0 * rows * d * f)      # six GEMMs of 2·rows·d·f flop each


def test_bound_selection(bench):
    c2 = bench.gemm_floors(768, 3072, 8, 16384, 2, PK)     # C2, N=1: long segments
    assert not c2["hbm_bound"] and c2["tensor_ms"] == pytest.approx(0.3293, rel=1e-3)
    c4 = bench.gemm_floors(1024, 4096, 32, 4096, 2, PK)    # C4 as a layer: ~128 rows per expert
    assert c4["hbm_bound"] and c4["hbm_ms"] > 1.9 * c4["tensor_ms"]
    # crossover: the ridge point of the pair of peaks (flop per byte) decides
    ridge = PK["bf16_sustained"] * 1e12 / (PK["hbm"] * 1e9)
    for rows in (512, 2048, 8192, 65536):
        fl = bench.gemm_floors(1024, 4096, 32, rows, 2, PK)
        assert fl["hbm_bound"] == (fl["flops"] / fl["bytes"] < ridge)
