"""Oracle for popularity-driven expert replication — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §5.2, Eq. (1):   n_e = N × Σ_t P(e) / N_t
"we adopt the first-fit-decreasing heuristic to pack them into the empty devices
so the total devices used are minimized"; experts without an estimate
"are assigned evenly to the remaining free devices if any; otherwise are randomly
assigned to a device"; the plan carries "how many tokens each
replica should handle to balance the load".

Readings (R14-R16): integer replica counts r_e = max(1, round-half-up(n_e)),
capped at N and trimmed largest-first (ties: larger expert id first) while
Σ r_e > N·max_per_device; a replica is an item of size n_e / r_e device-loads;
bins are devices of capacity 1.0 device-load and at most max_per_device experts;
an expert is never placed twice on one device.  Items are taken in (size desc,
expert id asc, replica asc) order and go to the lowest-id device where they fit
(first fit); an item that fits nowhere goes to the least-loaded eligible device
(lowest id on ties) — the deterministic stand-in for "randomly assigned" (R16).
Replica device lists are sorted ascending.  Token split (R14): the c tokens a
source rank s sends to expert e are cut, in slot order, into r_e contiguous
blocks whose sizes differ by at most 1 (the first c mod r_e blocks get one
extra); block q goes to replica (q + s) mod r_e.
"""
from __future__ import annotations

import math

EPS = 1e-9


class InfeasiblePlan(ValueError):
    """E > N × max_per_device, or a replica cannot be placed (SPEC S:381 error kind)."""


def replica_counts(popularity, num_devices: int, max_per_device: int):
    """Eq. (1) then integerisation (R15).  Returns (n_e list of float, r_e list of int)."""
    E = len(popularity)
    N = num_devices
    if E > N * max_per_device:
        raise InfeasiblePlan(f"{E} experts > {N} devices x {max_per_device} per device")
    n = [N * float(popularity[e]) for e in range(E)]
    r = [min(N, max(1, int(math.floor(n[e] + 0.5)))) for e in range(E)]
    while sum(r) > N * max_per_device:
        top = max(r)
        e = max(i for i in range(E) if r[i] == top)   # largest r_e; ties -> larger id
        r[e] -= 1
    return n, r


def place(popularity, num_devices: int, max_per_device: int):
    """First-fit-decreasing packing of replicas onto devices.

    Returns dict with replicas[E], replica_device[E][r_e] (ascending),
    hosted[N] (ascending expert ids), load[N] (device-loads)."""
    E = len(popularity)
    N = num_devices
    n, r = replica_counts(popularity, N, max_per_device)
    items = []
    for e in range(E):
        size = n[e] / r[e]
        for q in range(r[e]):
            items.append((size, e, q))
    items.sort(key=lambda it: (-it[0], it[1], it[2]))
    load = [0.0] * N
    hosted = [[] for _ in range(N)]
    for size, e, _ in items:
        eligible = [dv for dv in range(N) if len(hosted[dv]) < max_per_device and e not in hosted[dv]]
        if not eligible:
            raise InfeasiblePlan(f"no device can host another replica of expert {e}")
        fit = [dv for dv in eligible if load[dv] + size <= 1.0 + EPS]
        if fit:
            dv = fit[0]                                   # first fit
        else:
            dv = min(eligible, key=lambda v: (load[v], v))  # least loaded, lowest id
        load[dv] += size
        hosted[dv].append(e)
    replica_device = [sorted(dv for dv in range(N) if e in hosted[dv]) for e in range(E)]
    return {
        "replicas": r,
        "replica_device": replica_device,
        "hosted": [sorted(h) for h in hosted],
        "load": load,
        "n": n,
    }


def replica_split(count: int, replicas: int, source_rank: int):
    """Tokens of one (source, expert) pair per replica index (R14): list of length r_e."""
    base, extra = divmod(count, replicas)
    per_block = [base + (1 if q < extra else 0) for q in range(replicas)]
    out = [0] * replicas
    for q, c in enumerate(per_block):
        out[(q + source_rank) % replicas] += c
    return out


def route_counts(counts_per_source, plan, num_devices: int):
    """send[s][dv][e] = tokens source s sends to device dv for expert e under the plan."""
    S = len(counts_per_source)
    E = len(plan["replicas"])
    send = [[[0] * E for _ in range(num_devices)] for _ in range(S)]
    for s in range(S):
        for e in range(E):
            split = replica_split(int(counts_per_source[s][e]), plan["replicas"][e], s)
            for q, c in enumerate(split):
                send[s][plan["replica_device"][e][q]][e] += c
    return send
