"""Inference path with popularity-driven replication (S10) on one GPU: plan identical
to the oracle's, outputs equal to the oracle (dropless) and bitwise equal to the
static-placement training forward (P9)."""
import numpy as np
import pytest
import torch

import lina_inputs as li
from oracle import moe
from oracle import placement as oplace
from tests.parity_util import TOL, to_dev, tdtype

pytestmark = pytest.mark.gpu


def _run_infer(cfg, X, Wg, W1, W2, mpd, placement=None):
    import paper_2210_17223_b200 as lina
    comm = lina.Comm(1, 0, 0)
    dt = tdtype(cfg.dtype)
    T = X.shape[0]
    desc = lina.make_desc(T, cfg.d_model, cfg.d_ffn, cfg.num_experts, cfg.k, T, 1, dt)
    ws = torch.empty(lina.lina_moe_infer_workspace_size(comm, desc, mpd), dtype=torch.uint8, device="cuda")
    out = torch.empty((T, cfg.d_model), dtype=dt, device="cuda")
    plan = lina.lina_moe_infer_forward(comm, desc, to_dev(X, dt), to_dev(Wg, torch.float32), to_dev(W1, dt),
                                       to_dev(W2, dt), out, ws, placement=placement, max_per_device=mpd)
    torch.cuda.synchronize()
    return out.float().cpu().numpy(), plan


@pytest.mark.parametrize("family", ["zipf", "grid"])
def test_infer_single_gpu_matches_oracle_and_static(family):
    cfg = li.with_tokens(li.CONFIGS["C4"], 512)
    Wg, W1, W2 = li.layer_weights(cfg, 5, family)
    X, _ = li.layer_tokens(cfg, 5, 0, family, zipf_s=1.0)
    y, plan = _run_infer(cfg, X, Wg, W1, W2, mpd=cfg.num_experts)
    C = X.shape[0]  # dropless
    fw = moe.moe_forward([X], Wg, W1, W2, cfg.k, C, cfg.dtype)[0]
    assert moe.normwise_error(y, fw.y) <= TOL[cfg.dtype]
    pop = fw.counts / fw.counts.sum()
    ref = oplace.place(list(pop), 1, cfg.num_experts)
    assert plan.replicas == ref["replicas"] and plan.hosted == ref["hosted"]
    # P9: the static-placement training forward gives the same bits
    from tests.parity_util import gpu_layer
    if family == "grid":
        g = gpu_layer(cfg, 1, X, Wg, W1, W2, capacity=C)
        assert np.array_equal(g["y"], y)


@pytest.mark.parametrize("estimate_matches", [True, False])
def test_two_phase_keeps_or_replans(estimate_matches):
    """Phase two: a phase-one plan whose estimated top-2k experts equal the
    actual ones is used as given; otherwise the plan is re-computed from the actual
    popularity (= the oracle's placement of the batch histogram).  Output is the oracle's
    either way (the placement decides where experts run, not what they compute)."""
    import paper_2210_17223_b200 as lina
    from oracle import popularity as opop
    cfg = li.with_tokens(li.CONFIGS["C4"], 512)
    Wg, W1, W2 = li.layer_weights(cfg, 5, "zipf")
    X, _ = li.layer_tokens(cfg, 5, 0, "zipf", zipf_s=1.0)
    C = X.shape[0]
    fw = moe.moe_forward([X], Wg, W1, W2, cfg.k, C, cfg.dtype)[0]
    actual = fw.counts / fw.counts.sum()
    est = list(actual) if estimate_matches else list(actual[::-1])
    assert opop.phase_two(est, list(fw.counts), cfg.k) == estimate_matches
    E = cfg.num_experts
    given = oplace.place(est, 1, E)
    tables = lina.lina.PlacementTables(given["replicas"], given["replica_device"], given["hosted"])
    comm = lina.Comm(1, 0, 0)
    dt = tdtype(cfg.dtype)
    desc = lina.make_desc(C, cfg.d_model, cfg.d_ffn, E, cfg.k, C, 1, dt)
    ws = torch.empty(lina.lina_moe_infer_workspace_size(comm, desc, E), dtype=torch.uint8, device="cuda")
    out = torch.empty((C, cfg.d_model), dtype=dt, device="cuda")
    plan, replanned = lina.lina_moe_infer_forward_two_phase(
        comm, desc, to_dev(X, dt), to_dev(Wg, torch.float32), to_dev(W1, dt), to_dev(W2, dt), out, ws,
        tables, est)
    torch.cuda.synchronize()
    assert replanned == (not estimate_matches)
    ref = given if estimate_matches else oplace.place(list(actual), 1, E)
    assert plan.replicas == ref["replicas"] and plan.hosted == ref["hosted"]
    assert moe.normwise_error(out.float().cpu().numpy(), fw.y) <= TOL[cfg.dtype]


@pytest.mark.parametrize("bad,needle", [
    ({"replicas": [2, 1, 1, 1]}, "replicas 2 not in"),            # r_e > world (1)
    ({"replica_device": [[0], [5], [0], [0]]}, "not in [0, num_devices)"),
    ({"hosted": [[0, 1, 2, 7]]}, "not in [-1, num_experts)"),
    ({"hosted": [[0, 1, 2, -1]]}, "does not host it"),            # expert 3's device does not list it
    ({"hosted": [[0, 1, 2, 2]]}, "twice"),
])
def test_infer_rejects_inconsistent_placement(bad, needle):
    """A caller-supplied placement is checked entry by entry before its tables index device
    buffers: INVALID_ARGUMENT naming the violation, nothing launched."""
    import paper_2210_17223_b200 as lina
    from paper_2210_17223_b200.lina import LinaError, PlacementTables
    cfg = li.with_tokens(li.CONFIGS["C4"], 64, num_experts=4)
    Wg, W1, W2 = li.layer_weights(cfg, 5, "grid")
    X, _ = li.layer_tokens(cfg, 5, 0, "grid")
    tables = {"replicas": [1, 1, 1, 1], "replica_device": [[0], [0], [0], [0]], "hosted": [[0, 1, 2, 3]]}
    tables.update(bad)
    pl = PlacementTables(tables["replicas"], tables["replica_device"], tables["hosted"])
    with pytest.raises(LinaError) as ei:
        _run_infer(cfg, X, Wg, W1, W2, mpd=4, placement=pl)
    assert needle in str(ei.value) and ei.value.status == 1
