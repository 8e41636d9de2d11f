"""Phase-one estimation quality and cost on seeded Markov selection traces (host only).

For each (pattern strength p, path length l): profile a 50k-token training trace with the
native profiler (lina_popprof_*), then for 40 inference batches of 4096 tokens from the
same model estimate every layer m >= l and run the phase-two check against the batch's
actual selection counts.  Reports the top-2k accuracy ("if the top-2 ... estimated experts
are identical to the actual routing decision, we consider the estimation accurate",
PAPER.md §6.3.2), the fine-tune rate (= 1 - accuracy: phase two re-plans), the mean
max/mean device load of the estimate-based plan vs the actual-popularity plan, and the
host time of one estimate call and of one placement call (load = max/mean tokens per
device with each expert's actual tokens split evenly over its replicas).

    python tools/popularity_eval.py > profiles/r01_popularity_cpu.txt
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import lina_inputs as li  # noqa: E402
import paper_2210_17223_b200 as lina  # noqa: E402


def plan_load(plan, actual, N):
    """Max/mean device load when the actual tokens are split evenly over each expert's replicas."""
    load = np.zeros(N)
    for e, devs in enumerate(plan.replica_device):
        for dv in devs:
            load[dv] += actual[e] / len(devs)
    return load.max() / load.mean()


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=1)
    k = ap.parse_args().k
    E, L, N, T, MPD = 32, 6, 8, 4096, 8
    print(f"# E={E} experts, L={L} MoE layers, top-{k}, N={N} devices (max {MPD} experts each), "
          f"{T} tokens per inference batch, Zipf s=1.0 marginals, 50k-token profiling trace")
    print("#   p  l  accuracy  finetune  load(est plan)  load(actual plan)  load(static)  estimate ms  plan ms")
    for p in (0.3, 0.6, 0.9):
        for l in (1, 2, 3):
            train = li.selection_trace(50000, L, E, k, p, 1.0, seed=100)
            prof = lina.PopProfile(L, E, k, l)
            prof.add(train.sel)
            hits, n, le, la, ls, ms = 0, 0, [], [], [], []
            for b in range(40):
                batch = li.selection_trace(T, L, E, k, p, 1.0, seed=100, stream=1 + b,
                                           maps=train.maps, marginal=train.marginal)
                for m in range(l, L):
                    hist = np.ascontiguousarray(batch.sel[:, m - l:m, :])
                    t0 = time.perf_counter()
                    est, _ = prof.estimate(m, hist)
                    t1 = time.perf_counter()
                    plan = lina.lina_placement_compute(est, N, MPD)
                    t2 = time.perf_counter()
                    ms.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3))
                    actual = np.bincount(batch.sel[:, m, :].ravel(), minlength=E)
                    ok = lina.lina_phase_two_check(est, actual, k)
                    hits += ok
                    n += 1
                    le.append(plan_load(plan, actual, N))
                    la.append(plan_load(lina.lina_placement_compute(actual / actual.sum(), N, MPD), actual, N))
                    static = lina.lina_placement_compute([1.0 / E] * E, N, MPD)
                    ls.append(plan_load(static, actual, N))
            prof.close()
            print(f"{p:5.1f} {l:2d} {hits / n:9.3f} {1 - hits / n:9.3f} {np.mean(le):15.3f} "
                  f"{np.mean(la):18.3f} {np.mean(ls):13.3f} {np.median([a for a, _ in ms]):12.3f} "
                  f"{np.median([b for _, b in ms]):8.3f}")


if __name__ == "__main__":
    main()
