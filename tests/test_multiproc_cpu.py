"""Host-side logic of the N>1 path on CPU: two gloo processes play two ranks.

Each rank routes its own seeded tokens (the oracle's gate/top-k/capacity), allgathers
the per-expert counts, and computes the inference plan through the C ABI
(lina_placement_compute, lina_replica_split — pure host code, no GPU).  The ranks
must agree on the plan (no broadcast is used: DESIGN.md §7), it must equal the
oracle's, and the per-(source, device) token matrix must balance: what source s sends
to device dv for expert e is what dv expects from s, and every token goes to exactly
one replica.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import lina_inputs as li
    import paper_2210_17223_b200 as lina
    from oracle import moe
    from oracle import placement as oplace
    cfg = li.with_tokens(li.CONFIGS["C4"], 256, num_experts=8, d_model=64, d_ffn=256)
    Wg = li.gate_weight(cfg, 3, "zipf")
    X, _ = li.layer_tokens(cfg, 3, rank, "zipf", zipf_s=1.2)
    L = moe.gate_logits(X, Wg)
    idx = moe.top_k(L, cfg.k)
    _, counts = moe.capacity_slots(idx, cfg.num_experts, cfg.tokens_per_rank)
    allc = [torch.zeros(cfg.num_experts, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allc, torch.from_numpy(counts.astype(np.int64)))
    allc = np.stack([c.numpy() for c in allc])
    pop = allc.sum(0) / allc.sum()
    mpd = 2 * cfg.num_experts // world
    plan = lina.lina_placement_compute(list(pop), world, mpd)
    ref = oplace.place(list(pop), world, mpd)
    ok = plan.replicas == ref["replicas"] and plan.hosted == ref["hosted"] and \
        plan.replica_device == ref["replica_device"]
    # what I send to each device, per expert (R14 through the C ABI)
    send = np.zeros((world, cfg.num_experts), dtype=np.int64)
    for e in range(cfg.num_experts):
        split = lina.lina_replica_split(int(allc[rank, e]), plan.replicas[e], rank)
        for q_, n in enumerate(split):
            send[plan.replica_device[e][q_], e] += n
    ok &= bool((send.sum(0) == allc[rank]).all())
    # what each device expects from me: computed independently by every rank
    expect = np.zeros((world, world, cfg.num_experts), dtype=np.int64)
    for s in range(world):
        for e in range(cfg.num_experts):
            split = oplace.replica_split(int(allc[s, e]), plan.replicas[e], s)
            for q_, n in enumerate(split):
                expect[s, plan.replica_device[e][q_], e] += n
    ok &= bool((expect[rank] == send).all())
    plans = [None] * world
    dist.all_gather_object(plans, (plan.replicas, plan.replica_device, plan.hosted))
    ok &= all(p == plans[0] for p in plans)
    q.put((rank, ok, plan.replicas))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_plan_agreement_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29800 + os.getpid() % 100
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert all(min(r) >= 1 for _, _, r in res)


def _two_phase_worker(rank, world, port, q):
    """Phase one + phase two across two gloo ranks (§5.2): every rank
    profiles the same trace, estimates the next layer from ITS OWN tokens' paths,
    allgathers the estimates and the actual counts, and decides through the C ABI.  The
    ranks must reach the same phase-one plan, the same phase-two decision and the same
    final plan with no broadcast, each equal to the oracle's."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import lina_inputs as li
    import paper_2210_17223_b200 as lina
    from oracle import placement as oplace
    from oracle import popularity as opop
    E, L, k, l, m = 16, 5, 1, 2, 4
    train = li.selection_trace(20000, L, E, k, 0.8, 1.0, seed=9)          # shared profiling trace
    batch = li.selection_trace(1024, L, E, k, 0.8, 1.0, seed=9, stream=10 + rank,
                               maps=train.maps, marginal=train.marginal)  # this rank's tokens
    prof = lina.PopProfile(L, E, k, l)
    prof.add(train.sel)
    est_local, _ = prof.estimate(m, batch.sel[:, m - l:m, :])
    # phase one: the global estimate is the token-weighted mean of the ranks' estimates
    ests = [None] * world
    dist.all_gather_object(ests, est_local)
    est = [sum(e[x] for e in ests) / world for x in range(E)]
    mpd = E // world * 2
    plan1 = lina.lina_placement_compute(est, world, mpd)
    # phase two: actual counts after gating (here: the trace's layer-m selections)
    cnt = torch.from_numpy(np.bincount(batch.sel[:, m, :].ravel(), minlength=E).astype(np.int64))
    allc = [torch.zeros(E, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allc, cnt)
    actual = sum(c.numpy() for c in allc)
    same = lina.lina_phase_two_check(est, actual, k)
    final = plan1 if same else lina.lina_placement_compute(list(actual / actual.sum()), world, mpd)
    # the oracle, from the same inputs
    pf = opop.Profile(L, E, k, l)
    pf.add_trace(train.sel)
    ok = opop.estimate(pf, m, batch.sel[:, m - l:m, :])[0] == est_local
    ok &= same == opop.phase_two(est, list(actual), k)
    ref = oplace.place(est if same else list(actual / actual.sum()), world, mpd)
    ok &= final.replicas == ref["replicas"] and final.hosted == ref["hosted"]
    views = [None] * world
    dist.all_gather_object(views, (same, final.replicas, final.replica_device, final.hosted))
    ok &= all(v == views[0] for v in views)
    q.put((rank, bool(ok), bool(same)))
    dist.destroy_process_group()


def test_two_rank_two_phase_agreement_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 100
    procs = [ctx.Process(target=_two_phase_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
