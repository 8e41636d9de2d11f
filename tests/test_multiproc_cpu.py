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
