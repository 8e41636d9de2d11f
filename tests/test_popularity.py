"""Pins of oracle/popularity.py (sample-path profiles, phase-one estimate, phase-two check;
PAPER.md §5.2) — CPU only.

Each pin checks the oracle against something other than itself: the closed-form
next-layer distribution of the seeded Markov generator, analytic expectations,
hand-evaluated cases, and a brute-force regrouping of tiny traces.
"""
import itertools

import numpy as np
import pytest

import lina_inputs as li
from oracle import popularity as pop


def _profile(tr, l):
    T, L, k = tr.sel.shape
    pf = pop.Profile(L, tr.marginal.shape[1], k, l)
    pf.add_trace(tr.sel)
    return pf


def test_deterministic_map_gives_point_masses_and_exact_estimate():
    """p = 1, top-1: every Ψ is a point mass on the mapped expert, so the
    phase-one estimate of a fresh batch equals its actual next-layer histogram / N_t."""
    E, L = 8, 5
    tr = li.selection_trace(4000, L, E, 1, 1.0, 1.0, seed=3)
    for l in (1, 2, 3):
        pf = _profile(tr, l)
        for (m, s, path), c in pf.psi.items():
            a = path[-1][0]
            assert sum(c) == c[int(tr.maps[m - 1][a])], (m, s, path)
        fresh = li.selection_trace(500, L, E, 1, 1.0, 1.0, seed=3, stream=9, maps=tr.maps, marginal=tr.marginal)
        for m in range(l, L):
            est, picks = pop.estimate(pf, m, fresh.sel[:, m - l:m, :])
            actual = np.bincount(fresh.sel[:, m, 0], minlength=E) / 500.0
            assert np.array_equal(np.array(est), actual)
            assert [p[0] for p in picks] == list(fresh.sel[:, m, 0])


def test_independent_uniform_trace_is_uniform():
    """p = 0, Zipf s = 0 (independent uniform layers): every length-1 Ψ is within ±3pp of
    1/E at 50k tokens (analytic expectation; std ≈ 0.4pp per group here)."""
    E = 16
    tr = li.selection_trace(50000, 3, E, 1, 0.0, 0.0, seed=5)
    pf = _profile(tr, 1)
    for (m, s, path), c in pf.psi.items():
        psi = np.array(c) / sum(c)
        assert np.abs(psi - 1.0 / E).max() < 0.03


def test_markov_trace_reproduces_ground_truth_rows():
    """p = 0.6, Zipf 1.0, top-1: Ψ for path (a,) at layer m must approach the generator's
    closed form p·[e = map(a)] + (1-p)·marginal_m(e) (±2pp for groups of >= 2000 tokens)."""
    E, p = 8, 0.6
    tr = li.selection_trace(50000, 3, E, 1, p, 1.0, seed=11)
    pf = _profile(tr, 1)
    checked = 0
    for (m, s, path), c in pf.psi.items():
        if sum(c) < 2000:
            continue
        a = path[0][0]
        truth = (1 - p) * tr.marginal[m].copy()
        truth[int(tr.maps[m - 1][a])] += p
        assert np.abs(np.array(c) / sum(c) - truth).max() < 0.02, (m, a)
        checked += 1
    assert checked >= 4


def test_hand_evaluated_two_token_estimate():
    """Two tokens: A's path has Ψ = {e1: 0.5, e2: 0.5} (top-1 picks e1 by the id tie-break,
    P = 0.5), B's path has Ψ = {e1: 1.0} -> popularity(e1) = (0.5 + 1.0) / 2 = 0.75
    (the Σ_t P/N_t aggregation of Eq. (1))."""
    E = 4
    sel = np.array([[[0], [1]], [[0], [2]], [[3], [1]], [[3], [1]]], dtype=np.int32)   # [T=4, L=2, k=1]
    pf = pop.Profile(2, E, 1, 1)
    pf.add_trace(sel)
    est, picks = pop.estimate(pf, 1, [[[0]], [[3]]])
    assert est == [0.0, 0.75, 0.0, 0.0]
    assert picks == [[1], [1]]


def test_backoff_to_suffix_then_marginal():
    """R20: an unseen length-2 path uses its seen length-1 suffix; a token whose last
    expert was never seen before layer m uses layer m's marginal."""
    E = 4
    sel = np.array([[[0], [1], [2]], [[1], [1], [3]], [[2], [2], [0]]], dtype=np.int32)
    pf = pop.Profile(3, E, 1, 2)
    pf.add_trace(sel)
    # history (3, 1): path (3,1) unseen at m=2, suffix (1,) seen -> tokens 0,1 went to {2, 3}
    assert pf.distribution(2, [[3], [1]]) == [0, 0, 1, 1]
    # history (0, 0): neither (0,0) nor (0,) seen before layer 2 -> marginal of layer 2
    assert pf.distribution(2, [[0], [0]]) == [1, 0, 1, 1]
    est, _ = pop.estimate(pf, 2, [[[3], [1]]])
    assert est == [0.0, 0.0, 0.5, 0.0]       # tie {2, 3} -> lower id, Ψ = 1/2


def test_profile_brute_force_regrouping():
    """Ψ counts equal a brute-force regrouping: for every (layer, length, path) enumerate
    all expert-set tuples and count matching tokens with numpy masks (k = 2)."""
    E, L, k, l = 4, 4, 2, 2
    tr = li.selection_trace(60, L, E, k, 0.5, 0.5, seed=2)
    pf = _profile(tr, l)
    sets = [tuple(c) for c in itertools.combinations(range(E), k)]
    srt = np.sort(tr.sel, axis=2)
    n_keys = 0
    for m in range(1, L):
        for s in range(1, min(l, m) + 1):
            for path in itertools.product(sets, repeat=s):
                mask = np.ones(len(srt), dtype=bool)
                for q, el in enumerate(path):
                    mask &= (srt[:, m - s + q, :] == np.array(el)).all(axis=1)
                cnt = np.bincount(srt[mask, m, :].ravel(), minlength=E).tolist()
                key = (m, s, path)
                if mask.any():
                    assert pf.psi[key] == cnt
                    n_keys += 1
                else:
                    assert key not in pf.psi
    assert n_keys == len(pf.psi)


def test_k2_distribution_sums_to_one_and_popularity_bounded():
    """With top-2 gating Ψ sums to 1 (R20) and each token contributes at most 1 in total,
    so Σ_e popularity(e) <= 1 and N·popularity gives at most N devices (Eq. (1))."""
    tr = li.selection_trace(3000, 4, 8, 2, 0.6, 1.2, seed=4)
    pf = _profile(tr, 2)
    fresh = li.selection_trace(400, 4, 8, 2, 0.6, 1.2, seed=4, stream=3, maps=tr.maps, marginal=tr.marginal)
    for m in (2, 3):
        est, picks = pop.estimate(pf, m, fresh.sel[:, m - 2:m, :])
        assert 0.0 < sum(est) <= 1.0 + 1e-12
        assert all(len(p) == 2 for p in picks)


def test_layer_too_early_rejected():
    pf = pop.Profile(4, 4, 1, 3)
    with pytest.raises(ValueError):
        pop.estimate(pf, 2, [[[0], [1]]])


def test_phase_two_set_comparison():
    """identical top-2k lists -> no fine-tuning; order inside the list does not
    matter (R22); ties at rank 2k resolve to the lower expert id, deterministically."""
    k = 1
    assert pop.phase_two([0.5, 0.3, 0.1, 0.1], [10, 40, 0, 0], k)      # {0,1} vs {1,0}
    assert not pop.phase_two([0.5, 0.3, 0.1, 0.1], [10, 0, 40, 0], k)  # {0,1} vs {2,0}
    assert pop.top2k_set([0, 5, 5, 5], k) == frozenset({1, 2})           # tie at rank 2 -> id 2 < 3
    assert pop.top2k_set([0.25] * 4, 2) == frozenset({0, 1, 2, 3})


# ---------------------------------------------------------------------------------------
# The native implementation (liblina.so host functions, no GPU) against the oracle:
# bit-exact popularity (same fp64 operations in token order), identical top-k picks.
# ---------------------------------------------------------------------------------------

@pytest.fixture(scope="module")
def lina():
    import paper_2210_17223_b200 as pkg
    return pkg


@pytest.mark.parametrize("k,l,p,s", [(1, 1, 0.6, 1.0), (1, 3, 0.6, 1.2), (2, 2, 0.4, 0.8), (2, 3, 1.0, 0.0)])
def test_native_estimate_bit_exact(lina, k, l, p, s):
    E, L = 16, 6
    tr = li.selection_trace(3000, L, E, k, p, s, seed=21)
    pf = _profile(tr, l)
    nat = lina.PopProfile(L, E, k, l)
    nat.add(tr.sel[:1000])
    nat.add(tr.sel[1000:])                     # counts accumulate over calls
    fresh = li.selection_trace(700, L, E, k, p, s, seed=21, stream=5, maps=tr.maps, marginal=tr.marginal)
    for m in range(l, L):
        hist = fresh.sel[:, m - l:m, :]
        want, picks = pop.estimate(pf, m, hist)
        got, topk = nat.estimate(m, hist)
        assert got == want                      # bit-exact
        assert [list(r) for r in topk] == [list(q) if q else [-1] * k for q in picks]


@pytest.mark.parametrize("E,k,l", [(64, 2, 3), (64, 4, 3), (1024, 2, 3), (64, 10, 1)])
def test_native_packed_and_string_keys_agree_with_oracle(lina, E, k, l):
    """Paths are uint64 bit-packed keys when l·k·ceil(log2 E) <= 64 (E=64, k=2: 36 bits;
    E=1024, k=2: 60 bits) and byte strings otherwise (E=64, k=4: 72 bits): both layouts
    give the oracle's values bit-exactly."""
    L = 5
    tr = li.selection_trace(1500, L, E, k, 0.7, 1.0, seed=8)
    pf = _profile(tr, l)
    nat = lina.PopProfile(L, E, k, l)
    nat.add(tr.sel)
    fresh = li.selection_trace(300, L, E, k, 0.7, 1.0, seed=8, stream=2, maps=tr.maps, marginal=tr.marginal)
    for m in range(l, L):
        want, picks = pop.estimate(pf, m, fresh.sel[:, m - l:m, :])
        got, topk = nat.estimate(m, fresh.sel[:, m - l:m, :])
        assert got == want
        assert [list(r) for r in topk] == [list(q) if q else [-1] * k for q in picks]


def test_native_unseen_paths_and_empty_batch(lina):
    E = 4
    sel = np.array([[[0], [1], [2]], [[1], [1], [3]], [[2], [2], [0]]], dtype=np.int32)
    nat = lina.PopProfile(3, E, 1, 2)
    nat.add(sel)
    got, topk = nat.estimate(2, np.array([[[3], [1]], [[0], [0]]], dtype=np.int32))
    pf = pop.Profile(3, E, 1, 2)
    pf.add_trace(sel)
    want, _ = pop.estimate(pf, 2, [[[3], [1]], [[0], [0]]])
    assert got == want
    got0, _ = nat.estimate(2, np.zeros((0, 2, 1), dtype=np.int32))
    assert got0 == [0.0] * E
    empty = lina.PopProfile(3, E, 1, 2)           # nothing profiled: no distribution at all
    g, t = empty.estimate(2, np.array([[[0], [1]]], dtype=np.int32))
    assert g == [0.0] * E and t.tolist() == [[-1]]


def test_native_rejects_bad_arguments(lina):
    with pytest.raises(lina.LinaError) as ei:
        lina.PopProfile(1, 4, 5, 0)
    msg = str(ei.value)
    assert "num_layers" in msg and "k outside" in msg and "path_len" in msg
    nat = lina.PopProfile(3, 4, 1, 2)
    with pytest.raises(lina.LinaError):
        nat.add(np.array([[[0], [4], [1]]], dtype=np.int32))          # id outside [0, E)
    with pytest.raises(lina.LinaError):
        nat.estimate(1, np.zeros((1, 2, 1), dtype=np.int32))           # layer < path_len
    nat2 = lina.PopProfile(3, 4, 2, 1)
    with pytest.raises(lina.LinaError):
        nat2.add(np.array([[[0, 0], [1, 2], [1, 3]]], dtype=np.int32))  # expert twice in a layer


@pytest.mark.parametrize("seed", range(6))
def test_native_phase_two_matches_oracle(lina, seed):
    rng = np.random.default_rng(seed)
    E, k = 16, 1 + seed % 3
    for _ in range(50):
        est = rng.integers(0, 5, size=E) / 8.0           # many ties
        act = rng.integers(0, 6, size=E)
        assert lina.lina_phase_two_check(est, act, k) == pop.phase_two(list(est), list(act), k)
    assert lina.lina_phase_two_check([0.25] * 4, [1, 2, 3, 4], 2)   # 2k >= E: both lists are all experts


@pytest.mark.parametrize("E,k,l", [(16, 1, 3), (64, 4, 3)])      # packed keys / byte-string keys
def test_native_profile_save_load_round_trip(lina, tmp_path, E, k, l):
    """A profile built offline ("In the profiling stage") and saved gives, once
    loaded, the same estimates bit for bit; corrupt files are rejected with a reason."""
    L = 5
    tr = li.selection_trace(2000, L, E, k, 0.7, 1.0, seed=12)
    nat = lina.PopProfile(L, E, k, l)
    nat.add(tr.sel)
    path = str(tmp_path / "prof.bin")
    nat.save(path)
    back = lina.PopProfile.load(path)
    assert (back.L, back.E, back.k, back.l) == (L, E, k, l)
    fresh = li.selection_trace(300, L, E, k, 0.7, 1.0, seed=12, stream=4, maps=tr.maps, marginal=tr.marginal)
    for m in range(l, L):
        a, ta = nat.estimate(m, fresh.sel[:, m - l:m, :])
        b, tb = back.estimate(m, fresh.sel[:, m - l:m, :])
        assert a == b and (ta == tb).all()
    raw = open(path, "rb").read()
    for bad in (b"NOTAPROF" + raw[8:], raw[: len(raw) // 2]):
        open(path, "wb").write(bad)
        with pytest.raises(lina.LinaError):
            lina.PopProfile.load(path)
    with pytest.raises(lina.LinaError):
        lina.PopProfile.load(str(tmp_path / "missing.bin"))
