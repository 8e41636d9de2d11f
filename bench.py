"""Benchmark of the Lina B200 MoE layer: one step = forward + backward of the whole hot
path (gate, route, permute, dispatch all-to-all, expert FFN, combine all-to-all,
un-permute, and their backward) on synthetic tokens shaped like BASELINE.json's
configs[1] (GPT-2-small-shaped MoE layer: 8 experts, top-2, d_model 768, 8K
tokens per GPU, bf16).  Metric: MoE layer tokens/s fwd+bwd, whole job.

    python bench.py [--gpus N --steps K --warmup W] [--config C2] [--n-chunks n]
    python bench.py --impl reference ...      # the CPU oracle on a bounded sample

Multi-GPU: launched by torch.distributed.run, one rank per GPU (weak scaling: each
rank keeps T tokens; experts are partitioned E/N per rank).  Timing: CUDA events
on the launching stream around each step, L2 flushed (256 MB write) between
steps outside the events, barrier + synchronize on both sides, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
import lina_inputs as li  # noqa: E402

METRIC = "MoE layer tokens/s fwd+bwd"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="lina", choices=["lina", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(li.CONFIGS))
    ap.add_argument("--n-chunks", type=int, default=0,
                    help="0 = 1 (the fused transport needs no micro-op chunking; see DESIGN.md §7)")
    ap.add_argument("--nccl-ctas", type=int, default=8, help="ncclConfig_t.maxCTAs per communicator (N>1)")
    ap.add_argument("--family", default="balanced", choices=["balanced", "grid"])
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--copy-streams", type=int, default=1,
                    help="e2e: split each step's host<->device copies over this many streams per direction")
    ap.add_argument("--eager", action="store_true", help="launch every kernel from the host (no CUDA graph)")
    ap.add_argument("--cpu-sample", type=int, default=256, help="tokens in the oracle sample")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        p = json.load(open(path))
        return {"bf16_sustained": float(p["bf16_tflops_sustained"]), "bf16_burst": float(p["bf16_tflops"]),
                "hbm": float(p["hbm_gbs"]), "src": "measured"}
    except Exception:
        return {"bf16_sustained": 1400.0, "bf16_burst": 1590.0, "hbm": 6650.0, "src": "fallback"}


def gemm_floors(d, f, experts_local, kept, elt, pk):
    """Floors of the six expert GEMMs of one step; the bound is the higher.

    tensor: 12·d·f flop per kept assignment (fwd 4df, bwd 8df) at the sustained bf16 peak.
    HBM: the algorithmic bytes of the six GEMMs as separate kernels at the measured copy
    bandwidth — each local expert's W1 and W2 read twice (GEMM1/GEMM2, the two dgrads) and
    dW1, dW2 written once (6·d·f elements per expert); per kept row 6·d + 6·f activation
    elements (X, H, Y, dY, dH, dX in and out, and the wgrads' two operands each) and the
    ReLU' bits written and read once (2·f/8 bytes).
    """
    flops = 12.0 * kept * d * f
    nbytes = 6.0 * experts_local * d * f * elt + kept * (6.0 * (d + f) * elt + 2.0 * f / 8)
    t_tensor = flops / (pk["bf16_sustained"] * 1e12) * 1e3
    t_hbm = nbytes / (pk["hbm"] * 1e9) * 1e3
    return {"flops": flops, "bytes": nbytes, "tensor_ms": t_tensor, "hbm_ms": t_hbm, "hbm_bound": t_hbm > t_tensor}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------- CPU oracle timing


def oracle_step_sample(cfg, seed, family, sample_tokens, world):
    """One oracle fwd+bwd over a bounded sample: `sample_tokens` tokens of one rank, all experts.
    Returns (seconds, tokens)."""
    from oracle import moe
    sub = li.with_tokens(cfg, sample_tokens)
    Wg, W1, W2 = li.layer_weights(sub, seed, family)
    X, dY = li.layer_tokens(sub, seed, 0, family)
    C = li.with_tokens(cfg, sample_tokens).capacity()
    t0 = time.perf_counter()
    fw = moe.moe_forward([X], Wg, W1, W2, cfg.k, C, cfg.dtype)
    moe.moe_backward(fw, [X], [dY], Wg, W1, W2, cfg.k, cfg.dtype)
    return time.perf_counter() - t0, sample_tokens


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        n = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
        return int(n)
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = li.CONFIGS[args.config]
    for _ in range(args.warmup):
        oracle_step_sample(cfg, args.seed, args.family, args.cpu_sample, world)
    tot, toks = 0.0, 0
    for _ in range(args.steps):
        s, n = oracle_step_sample(cfg, args.seed, args.family, args.cpu_sample, world)
        tot += s
        toks += n
    value = toks / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: E={cfg.num_experts} top-{cfg.k} d={cfg.d_model} f={cfg.d_ffn} "
                               f"T/rank={cfg.tokens_per_rank} cf={cfg.cf} {cfg.dtype}",
                   "sample_tokens": args.cpu_sample},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cpu_threads(), "kind": "oracle",
                         "sample": f"{args.cpu_sample} tokens of one rank's {cfg.name} batch, fwd+bwd, all experts, "
                                   "fp64 numpy oracle (per step)"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.gpus != world and world == 1 and args.gpus > 1:
        print(f"--gpus {args.gpus} needs torch.distributed.run with {args.gpus} processes", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        return run_reference(args)

    import paper_2210_17223_b200 as lina

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
        uid = [lina.lina_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = lina.Comm(world, rank, local, uid[0], args.nccl_ctas)
    else:
        comm = lina.Comm(1, 0, local)

    cfg = li.CONFIGS[args.config]
    T, d, f, E, k = cfg.tokens_per_rank, cfg.d_model, cfg.d_ffn, cfg.num_experts, cfg.k
    C = cfg.capacity()
    El = E // world
    n_chunks = args.n_chunks or 1
    transport = os.environ.get("LINA_TRANSPORT", "fused") if world > 1 else "none"
    tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    Wg_np, W1_np, W2_np = li.layer_weights(cfg, args.seed, args.family, experts=range(rank * El, (rank + 1) * El))
    X_np, dY_np = li.layer_tokens(cfg, args.seed, rank, args.family)
    wg = torch.from_numpy(Wg_np).to(dev)
    w1 = torch.from_numpy(W1_np).to(tdt).to(dev)
    w2 = torch.from_numpy(W2_np).to(tdt).to(dev)
    x = torch.from_numpy(X_np).to(tdt).to(dev)
    dy = torch.from_numpy(dY_np).to(tdt).to(dev)
    del W1_np, W2_np
    layer = lina.MoELayer(comm, T, d, f, E, k, C, n_chunks, tdt, dev)
    outs = {"y": torch.empty((T, d), dtype=tdt, device=dev), "dx": torch.empty((T, d), dtype=tdt, device=dev),
            "dwg": torch.empty_like(wg), "dw1": torch.empty_like(w1), "dw2": torch.empty_like(w2)}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step(xx, dyy):
        layer.forward(xx, wg, w1, w2, out=outs["y"])
        layer.backward(dyy, xx, wg, w1, w2, outs["dx"], outs["dwg"], outs["dw1"], outs["dw2"])

    # routing of this batch (identical every step): kept assignments for the algorithmic flop count
    layer.forward(x, wg, w1, w2, out=outs["y"], want_route=True)
    counts = layer.route_t["counts"].cpu().numpy()
    kept_local = int(np.minimum(counts, C).sum())
    for _ in range(args.warmup):
        step(x, dy)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    # ---------------- one step captured as a CUDA graph: the timed loop replays it (the
    # library is stream-ordered, host-sync free and keeps its cross-rank rounds in device
    # memory, so a replay is a full step); --eager launches every kernel from the host
    def capture(xx, dyy, yy, dxx):
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            layer.forward(xx, wg, w1, w2, out=yy)
            layer.backward(dyy, xx, wg, w1, w2, dxx, outs["dwg"], outs["dw1"], outs["dw2"])
        torch.cuda.synchronize()
        return g

    launch_mode = "eager"
    graph = None
    if not args.eager:
        try:
            barrier()
            graph = capture(x, dy, outs["y"], outs["dx"])
            barrier()
            graph.replay()
            torch.cuda.synchronize()
            launch_mode = "cuda graph (one replay per step)"
        except Exception as exc:  # noqa: BLE001 - report and time the eager path instead
            graph = None
            launch_mode = f"eager (graph capture failed: {type(exc).__name__})"
            torch.cuda.synchronize()
    run_step = graph.replay if graph is not None else (lambda: step(x, dy))

    # ---------------- timed region (device time, per-step events, L2 flushed between steps)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        h0 = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record(stream)
            run_step()
            evs[i][1].record(stream)
        host_ms = (time.perf_counter() - h0) * 1e3 / args.steps  # enqueue time per step (diagnostic)
        torch.cuda.synchronize()
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = float(sum(step_ms))

    # ---------------- the same steps launched eagerly with the library's GEMM-phase events
    # (roofline numerator) and launch counter (gpu_launches); not part of `value`
    lina.lina_profile_read(comm)
    lina.lina_profile_enable(comm, True)
    barrier()
    torch.cuda.synchronize()
    evs_e = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        evs_e[i][0].record(stream)
        step(x, dy)
        evs_e[i][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    lina.lina_profile_enable(comm, False)
    prof = lina.lina_profile_read(comm)
    gemm_ms = prof["gemm_ms"]
    eager_ms = torch.tensor([sum(a.elapsed_time(b) for a, b in evs_e) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(eager_ms, op=torch.distributed.ReduceOp.MAX)
    eager_step_ms = float(eager_ms[0])
    t_all = torch.tensor([total_ms, gemm_ms, float(kept_local)], dtype=torch.float64, device=dev)
    if world > 1:
        mx = t_all.clone()
        torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
        sm = t_all.clone()
        torch.distributed.all_reduce(sm, op=torch.distributed.ReduceOp.SUM)
        total_ms_max, kept_total = float(mx[0]), float(sm[2])
    else:
        total_ms_max, kept_total = total_ms, float(kept_local)
    value = world * T * args.steps / (total_ms_max / 1e3)

    # ---------------- exposed communication (N>1): compute-only and all-to-all-only passes
    a2a = None
    if world > 1:
        def timed(flags):
            lina.lina_profile_enable(comm, flags)
            barrier()
            torch.cuda.synchronize()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)]
            for i in range(args.steps):
                flush.zero_()
                ev[i][0].record(stream)
                step(x, dy)
                ev[i][1].record(stream)
            torch.cuda.synchronize()
            barrier()
            lina.lina_profile_enable(comm, 0)
            lina.lina_profile_read(comm)
            t = torch.tensor([sum(a.elapsed_time(b) for a, b in ev) / args.steps], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            return float(t[0])
        t_comp = timed(2)
        t_comm = timed(4)
        t_step = eager_step_ms  # the compute-only and collectives-only passes are eager too
        exposed = max(0.0, t_step - t_comp)
        from paper_2210_17223_b200.lina import LINA_BF16  # noqa: F401
        elt = 2 if tdt == torch.bfloat16 else 4
        import math
        cm_rows = C if n_chunks == 1 else None
        if cm_rows is None:  # chunk pitch (R10)
            base = math.ceil(C / n_chunks)
            cm_rows = base
            for al in (256, 128, 64):
                cmv = math.ceil(base / al) * al
                if (n_chunks - 1) * cmv < C:
                    cm_rows = cmv
                    break
        bytes_rank = 4 * n_chunks * E * cm_rows * d * elt   # 4 all-to-alls of the padded send buffer
        algbw = bytes_rank / (t_comm / 1e3) / 1e9
        a2a = {"ms_per_step_isolated": t_comm,
               # the fused transport has no stand-alone collective: its isolated pass moves the
               # same bytes with the copy-engine transport
               "isolated_transport": "ce" if transport == "fused" else transport,
               "ms_per_step_compute_only": t_comp, "ms_per_step_eager": t_step,
               "exposed_ms_per_step": exposed,
               "hidden_frac": (1.0 - exposed / t_comm) if t_comm > 0 else None,
               "algbw_GBps": algbw, "busbw_GBps": algbw * (world - 1) / world,
               "bytes_per_rank_per_step": bytes_rank, "nccl_max_ctas": args.nccl_ctas}

    # ---------------- end to end through the public API, host buffers (pinned), copies timed
    # Every step copies its inputs (x, dY) from pinned host memory and its results (y, dX)
    # back to pinned host memory inside the timed region.  The copies run on two copy
    # streams, double-buffered, so step i+1's inputs and step i-1's results move while
    # step i computes (the way a training input pipeline feeds the layer).
    e2e = None
    if not args.no_e2e:
        xp = torch.from_numpy(X_np).to(tdt).pin_memory()
        dyp = torch.from_numpy(dY_np).to(tdt).pin_memory()
        yp = [torch.empty((T, d), dtype=tdt).pin_memory() for _ in range(2)]
        dxp = [torch.empty((T, d), dtype=tdt).pin_memory() for _ in range(2)]
        xd = [torch.empty_like(x) for _ in range(2)]
        dyd = [torch.empty_like(dy) for _ in range(2)]
        yd = [torch.empty_like(outs["y"]) for _ in range(2)]
        dxd = [torch.empty_like(outs["dx"]) for _ in range(2)]
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        in_ready = [torch.cuda.Event() for _ in range(2)]
        comp_done = [torch.cuda.Event() for _ in range(2)]
        out_done = [torch.cuda.Event() for _ in range(2)]
        nsplit = max(1, args.copy_streams)
        # extra streams per direction (nsplit > 1): row slices of every copy run on them
        x_in = [torch.cuda.Stream(dev) for _ in range(nsplit - 1)]
        x_out = [torch.cuda.Stream(dev) for _ in range(nsplit - 1)]

        def split_copy(main, extra, pairs):
            """Copy (dst, src) pairs on `main`, or as row slices over main + extra streams."""
            if not extra:
                for dst, src in pairs:
                    dst.copy_(src, non_blocking=True)
                return
            ev = torch.cuda.Event()
            ev.record(main)
            streams = [main] + extra
            for st in extra:
                st.wait_event(ev)
            rows = -(-T // len(streams))
            for q, st in enumerate(streams):
                with torch.cuda.stream(st):
                    for dst, src in pairs:
                        dst[q * rows:(q + 1) * rows].copy_(src[q * rows:(q + 1) * rows], non_blocking=True)
            for st in extra:
                main.wait_stream(st)

        def fetch(i):
            b = i % 2
            with torch.cuda.stream(s_in):
                if i >= 2:
                    s_in.wait_event(comp_done[b])  # step i-2 is done reading this buffer
                split_copy(s_in, x_in, [(xd[b], xp), (dyd[b], dyp)])
                in_ready[b].record(s_in)

        e2e_graphs = None
        if graph is not None:  # the same step graph, one per buffer set
            barrier()
            e2e_graphs = [capture(xd[b], dyd[b], yd[b], dxd[b]) for b in range(2)]
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s_in.wait_stream(stream)
        s_out.wait_stream(stream)
        fetch(0)
        for i in range(args.steps):
            b = i % 2
            if i + 1 < args.steps:
                fetch(i + 1)
            stream.wait_event(in_ready[b])
            if i >= 2:
                stream.wait_event(out_done[b])  # step i-2's results have left yd[b] / dxd[b]
            if e2e_graphs:
                e2e_graphs[b].replay()
            else:
                layer.forward(xd[b], wg, w1, w2, out=yd[b])
                layer.backward(dyd[b], xd[b], wg, w1, w2, dxd[b], outs["dwg"], outs["dw1"], outs["dw2"])
            comp_done[b].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(comp_done[b])
                split_copy(s_out, x_out, [(yp[b], yd[b]), (dxp[b], dxd[b])])
                out_done[b].record(s_out)
        stream.wait_stream(s_out)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(e2e_ms, op=torch.distributed.ReduceOp.MAX)
        elt = 2 if tdt == torch.bfloat16 else 4
        e2e = {"value": world * T * args.steps / (float(e2e_ms[0]) / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": 2 * T * d * elt, "d2h_bytes_per_step": 2 * T * d * elt,
               "copies": "pinned host <-> device, double-buffered, overlapping compute, "
                         f"{nsplit} stream(s) per direction"}

    # ---------------- roofline of the dominant kernel family (the six expert GEMMs)
    pk = peaks()
    fl = gemm_floors(d, f, E // world, kept_local, 2 if tdt == torch.bfloat16 else 4, pk)
    flops_per_step_local, bytes_per_step_local = fl["flops"], fl["bytes"]
    t_tensor_ms, t_hbm_ms, hbm_bound = fl["tensor_ms"], fl["hbm_ms"], fl["hbm_bound"]
    gemm_ms_per_step = gemm_ms / max(args.steps, 1)
    if hbm_bound:
        achieved = bytes_per_step_local / (gemm_ms_per_step / 1e3) / 1e9 if gemm_ms > 0 else None
        peak, unit, psrc = pk["hbm"], "GB/s", f"{pk['src']} HBM copy bandwidth (MEASURED_PEAKS.json)"
    else:
        achieved = flops_per_step_local / (gemm_ms_per_step / 1e3) / 1e12 if gemm_ms > 0 else None
        peak, unit, psrc = pk["bf16_sustained"], "TFLOP/s", f"{pk['src']} bf16 sustained (MEASURED_PEAKS.json)"
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.config)
        except Exception:
            traffic = None
    roof = {"bound": "hbm" if hbm_bound else "tensor",
            "kernel": "expert grouped GEMMs (fwd GEMM1+ReLU, GEMM2; bwd dgrad x2, wgrad x2)",
            "achieved": achieved, "peak": peak, "unit": unit,
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "peak_src": psrc,
            "gemm_ms_per_step": gemm_ms_per_step,
            "gemm_share_of_step": gemm_ms_per_step / (total_ms / args.steps) if total_ms > 0 else None,
            "algorithmic_flops_per_step": flops_per_step_local,
            "algorithmic_bytes_per_step": bytes_per_step_local,
            "floors_ms": {"tensor": t_tensor_ms, "hbm": t_hbm_ms}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        s, n = oracle_step_sample(cfg, args.seed, args.family, args.cpu_sample, world)
        cpu = {"value": n / s, "unit": "tokens/s", "cores": cpu_threads(), "kind": "oracle",
               "sample": f"{n} tokens of the {cfg.name} batch, fwd+bwd, all {E} experts, fp64 numpy oracle "
                         f"({s:.2f} s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16" if tdt == torch.bfloat16 else "f32",
            "data": f"synthetic ({args.family} family, seeded random-init weights)",
            "config": {"workload": f"{cfg.name}: E={E} top-{k} d={d} f={f} T/rank={T} cf={cfg.cf} C={C} "
                                   f"n_chunks={n_chunks} {cfg.dtype}",
                       "global_batch": world * T, "parallelism": f"ep{world}", "a2a_transport": transport,
                       "l2": "flushed between timed steps (256 MB write, outside the step events)",
                       "launch": launch_mode,
                       "kept_assignments": int(kept_total)},
            "roofline": roof,
            "a2a": a2a,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(prof["kernel_launches"]),  # this library's kernels per K steps (eager count)
            "clocks": clocks.summary(),
            "step_ms": {"min": min(step_ms), "median": float(np.median(step_ms)), "max": max(step_ms)},
            "host_enqueue_ms_per_step": host_ms,
        }
        print(json.dumps(line), flush=True)
    comm.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
