"""CPU-side checks of the C ABI: the library loads, exports every declared symbol,
and its host-only entry points (placement, replica split, argument validation)
agree with the oracle / the header's contract.  No GPU compute is called."""
import os
import re

import numpy as np
import pytest

from oracle import placement as oplace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "lina.h")).read()
    return sorted(set(re.findall(r"^\s*(?:lina_status|const char\*)\s+(lina_\w+)\s*\(", hdr, re.M)))


@pytest.fixture(scope="module")
def lina():
    import paper_2210_17223_b200 as pkg
    return pkg


def test_library_exports_every_declared_symbol(lina):
    lib = lina.load()
    declared = _declared_symbols()
    assert len(declared) >= 18
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(lina.ABI_SYMBOLS) == declared


def test_version(lina):
    assert "sm_100a" in lina.lina_version()


def test_comm_init_without_gpu_is_unsupported(lina):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(lina.LinaError) as ei:
        lina.Comm(1, 0, 0)
    assert ei.value.status == 2          # LINA_ERR_UNSUPPORTED: no CPU fallback


def test_comm_init_lists_every_violation(lina):
    with pytest.raises(lina.LinaError) as ei:
        lina.Comm(world=0, rank=3, device=0, unique_id=None, nccl_max_ctas=-1)
    msg = str(ei.value)
    assert ei.value.status == 1
    for frag in ["world < 1", "rank not in", "nccl_max_ctas < 0"]:
        assert frag in msg


def _golden_placements(golden_dir):
    import json
    return json.load(open(os.path.join(golden_dir, "placement_cases.json")))["cases"]


def test_placement_golden_through_abi(lina, golden_dir):
    for c in _golden_placements(golden_dir):
        t = lina.lina_placement_compute(c["popularity"], c["N"], c["max_per_device"])
        assert t.replicas == c["replicas"]
        assert t.hosted == c["hosted"]


@pytest.mark.parametrize("seed", range(40))
def test_placement_matches_oracle_bit_exact(lina, seed):
    rng = np.random.default_rng(700 + seed)
    N = int(rng.integers(1, 9)); mpd = int(rng.integers(1, 9))
    E = int(rng.integers(1, N * mpd + 1))
    pop = rng.dirichlet(np.full(E, 0.4))
    if seed % 3 == 0:
        pop[rng.random(E) < 0.3] = 0.0
    pop = list(pop)
    ref = oplace.place(pop, N, mpd)
    got = lina.lina_placement_compute(pop, N, mpd)
    assert got.replicas == ref["replicas"]
    assert got.replica_device == ref["replica_device"]
    assert got.hosted == ref["hosted"]


def test_placement_zipf_c4_worked_case(lina):
    """C4 reading (SURVEY.md §8(c) Q15 notes): E=32, N=8, Zipf s=1.0 -> n_0 = 1.97 -> r_0 = 2."""
    import lina_inputs as li
    pop = li.zipf_probs(32, 1.0)
    t = lina.lina_placement_compute(list(pop), 8, 8)
    assert t.replicas[0] == 2
    assert sum(t.replicas) == sum(oplace.place(list(pop), 8, 8)["replicas"])


def test_placement_infeasible(lina):
    with pytest.raises(lina.LinaError) as ei:
        lina.lina_placement_compute([0.1] * 10, 2, 4)
    assert ei.value.status == 3


@pytest.mark.parametrize("count,r,s", [(0, 1, 0), (7, 3, 0), (7, 3, 1), (100, 7, 5), (5, 8, 3)])
def test_replica_split_matches_oracle(lina, count, r, s):
    assert lina.lina_replica_split(count, r, s) == oplace.replica_split(count, r, s)


def test_product_path_does_not_import_oracle():
    """The product package must never reach the oracle (no CPU fallback)."""
    pkg_dir = os.path.join(ROOT, "paper_2210_17223_b200")
    for dp, _, files in os.walk(pkg_dir):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".h")):
                src = open(os.path.join(dp, f), errors="ignore").read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_two_phase_rejects_missing_phase_one_inputs(lina):
    """lina_moe_infer_forward_two_phase needs the phase-one plan and the estimate; the
    check happens before any device work (no GPU needed)."""
    import ctypes
    lib = lina.load()
    E = 4
    est = (ctypes.c_double * E)(*([0.25] * E))
    st = lib.lina_moe_infer_forward_two_phase(None, None, None, None, None, None, None, None, est,
                                              None, None, None, 0, None)
    assert st == 1 and b"placement" in lib.lina_last_error()
    pl = lina.lina._alloc_placement(E, 1, E)
    st = lib.lina_moe_infer_forward_two_phase(None, None, None, None, None, None, None, ctypes.byref(pl), None,
                                              None, None, None, 0, None)
    assert st == 1 and b"host_estimated" in lib.lina_last_error()
