"""Benchmark of the Lina B200 MoE layer: one step = forward + backward of the whole hot
path (gate, route, permute, dispatch all-to-all, expert FFN, combine all-to-all,
un-permute, and their backward; at N > 1 also the gate-weight gradient allreduce
through the micro-op scheduler) on synthetic tokens shaped like BASELINE.json's
configs[4] (the scale sweep "at 1/2/4/8 B200": 64 experts, top-2, d_model 2048,
d_ffn 8192, 32K tokens per GPU, bf16) — the largest single-GPU configuration and the
one the metric's "at 1/2/4/8 B200" names.  Metric: MoE layer tokens/s fwd+bwd,
whole job.

    python bench.py [--gpus N --steps K --warmup W] [--config C5] [--n-chunks n]
    python bench.py --impl reference ...      # the CPU oracle on a bounded sample
    torchrun ... bench.py --gpus N --sweep-chunks 1,2,4,8   # H(n) per micro-op count

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
import threading
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
    ap.add_argument("--config", default="C5", choices=sorted(li.CONFIGS))
    ap.add_argument("--n-chunks", type=int, default=0,
                    help="0 = 1 (the fused transport needs no micro-op chunking; see DESIGN.md §7)")
    ap.add_argument("--nccl-ctas", type=int, default=8, help="ncclConfig_t.maxCTAs per communicator (N>1)")
    ap.add_argument("--family", default="balanced", choices=["balanced", "grid"])
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--copy-streams", type=int, default=2,
                    help="e2e: split each step's host<->device copies over this many streams per direction")
    ap.add_argument("--eager", action="store_true", help="launch every kernel from the host (no CUDA graph)")
    ap.add_argument("--cpu-sample", type=int, default=0,
                    help="tokens in the oracle sample (0 = 64 for C5, 256 otherwise: ~10-30 s of host work)")
    ap.add_argument("--sweep-chunks", default="",
                    help="N > 1: comma list of n_chunks; H(n) and the pipelining efficiency for each (eager passes)")
    ap.add_argument("--sched-policy", default="lina", choices=["lina", "baseline", "naive", "defer"],
                    help="N > 1: allreduce scheduler policy for the per-step dWg allreduce")
    a = ap.parse_args()
    if a.cpu_sample <= 0:
        a.cpu_sample = 64 if a.config == "C5" else 256
    return a


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def progress(msg):
    """Phase markers on stderr (rank 0) — a hung multi-rank run shows where it stopped."""
    if int(os.environ.get("RANK", "0")) == 0:
        print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        p = json.load(open(path))
        return {"bf16_sustained": float(p["bf16_tflops_sustained"]), "bf16_burst": float(p["bf16_tflops"]),
                "hbm": float(p["hbm_gbs"]), "src": "measured"}
    except Exception:
        return {"bf16_sustained": 1400.0, "bf16_burst": 1590.0, "hbm": 6650.0, "src": "fallback"}


def choose_peak(pk, clk):
    """Burst bf16 peak unless the timed region ran power-capped or with its median SM clock
    well below max (then the sustained peak, measured at a loaded clock, is the fair one)."""
    reasons = clk.get("reasons") or []
    sm, mx = clk.get("sm_mhz"), clk.get("sm_max_mhz")
    low = sm is not None and mx and sm < 0.9 * mx
    if "sw_power_cap" in reasons or low:
        why = "sw_power_cap" if "sw_power_cap" in reasons else f"median SM clock {sm:.0f} < 0.9 x {mx:.0f} MHz"
        return pk["bf16_sustained"], "sustained", why
    why = (f"median SM clock {sm:.0f} of {mx:.0f} MHz, no power cap" if sm is not None
           else "no clock record (nvidia-smi unavailable)")
    return pk["bf16_burst"], "burst", why


def layer_floor(d, f, E_local, k, T, kept, P, elt, tc_tflops, hbm_gbs, nvlink_gbs=900.0):
    """SURVEY.md §8(d) layer roofline of one fwd+bwd step on one rank:
    t_roof = max(F_gemm / TC, B_a2a,offGPU / NVLink) + B_memkernels / HBM.

    F_gemm = 12·k·d·f per kept assignment; B_a2a per direction = the 4 all-to-alls' kept rows
    (d·elt each) × (P−1)/P leaving the GPU; B_memkernels = the HBM-bound kernels' algorithmic
    bytes per token: forward d·elt·(3 + 2k) (gate reads X; permute reads X, writes k rows;
    combine reads k rows, writes y) and backward d·elt·(3 + 3k) (combine-backward reads dY and
    k output rows, writes k rows; dX reads k rows, writes dX; dWg reads X)."""
    flops = 12.0 * kept * d * f
    a2a_dir = 4.0 * kept * d * elt * (P - 1) / P
    mem = T * d * elt * ((3 + 2 * k) + (3 + 3 * k))
    t_gemm = flops / (tc_tflops * 1e12) * 1e3
    t_a2a = a2a_dir / (nvlink_gbs * 1e9) * 1e3
    t_mem = mem / (hbm_gbs * 1e9) * 1e3
    return {"t_roof_ms": max(t_gemm, t_a2a) + t_mem, "t_gemm_ms": t_gemm, "t_a2a_ms": t_a2a, "t_mem_ms": t_mem,
            "gemm_flops": flops, "a2a_bytes_per_direction": a2a_dir, "memkernel_bytes": mem}


def gemm_floors(d, f, experts_local, kept, elt, pk, tc_tflops):
    """Floors of the six expert GEMMs of one step; the bound is the higher.

    tensor: 12·d·f flop per kept assignment (fwd 4df, bwd 8df) at the chosen bf16 peak.
    HBM: the algorithmic bytes of the six GEMMs as separate kernels at the measured copy
    bandwidth — each local expert's W1 and W2 read twice (GEMM1/GEMM2, the two dgrads) and
    dW1, dW2 written once (6·d·f elements per expert); per kept row 6·d + 6·f activation
    elements (X, H, Y, dY, dH, dX in and out, and the wgrads' two operands each) and the
    ReLU' bits written and read once (2·f/8 bytes).
    """
    flops = 12.0 * kept * d * f
    nbytes = 6.0 * experts_local * d * f * elt + kept * (6.0 * (d + f) * elt + 2.0 * f / 8)
    t_tensor = flops / (tc_tflops * 1e12) * 1e3
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
        # Returns once nvidia-smi has produced its first sample: its NVML start-up takes driver
        # locks that stall concurrent CUDA calls for tens of ms (at N > 1 the host-issued dWg
        # allreduce of a step waited behind it: one 24-28 ms step in a 20-step region), so it
        # must be done before the timed region starts.
        self.lines = []
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        if self.proc is not None:
            self.reader = threading.Thread(target=self._read, daemon=True)
            self.reader.start()
            t0 = time.perf_counter()
            while not self.lines and time.perf_counter() - t0 < 10 and self.proc.poll() is None:
                time.sleep(0.02)
            time.sleep(0.2)
        return self

    def _read(self):
        for line in self.proc.stdout:
            if line.strip():
                self.lines.append(line)

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=10)
            except Exception:
                self.proc.kill()
            self.reader.join(timeout=5)

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


def oracle_sample_inputs(cfg, seed, family, sample_tokens):
    """The gate weight, `sample_tokens` tokens of one rank and the expert weights, fp64, built
    outside any timing.  The expert weight arrays have all E experts (np.zeros: untouched pages
    cost no memory) with the experts the sample's tokens select filled in — the layer reads no
    other expert (C5: 17 GB of fp64 weights for all 64, more than a 62 GB host holds next to
    the oracle's gradients)."""
    from oracle import moe
    sub = li.with_tokens(cfg, sample_tokens)
    Wg = li.gate_weight(sub, seed, family)
    X, dY = li.layer_tokens(sub, seed, 0, family)
    used = sorted(set(int(e) for e in moe.top_k(moe.gate_logits(X, Wg), cfg.k).ravel()))
    W1 = np.zeros((cfg.num_experts, cfg.d_ffn, cfg.d_model))
    W2 = np.zeros((cfg.num_experts, cfg.d_model, cfg.d_ffn))
    for e in used:
        W1[e], W2[e] = li.expert_weights(sub, seed, e, family)
    return Wg, W1, W2, X, dY


def oracle_step_sample(cfg, seed, family, sample_tokens, world, inputs=None):
    """One oracle fwd+bwd over a bounded sample: `sample_tokens` tokens of one rank, all experts.
    Returns (seconds, tokens)."""
    from oracle import moe
    Wg, W1, W2, X, dY = inputs if inputs is not None else oracle_sample_inputs(cfg, seed, family, sample_tokens)
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
    # the sample's inputs are generated once (C5: up to 17 GB of fp64 expert weights, ~20 s); a
    # step is the oracle's fwd+bwd over them.  At C5 a step costs ~25-80 s whatever the token
    # count: the oracle zero-fills and rounds to bf16 the weight gradients of all 64 experts
    # (2 x 64 x 16.8 M values) — the oracle as it stands is not tuned for this
    inputs = oracle_sample_inputs(cfg, args.seed, args.family, args.cpu_sample)
    for _ in range(args.warmup):
        oracle_step_sample(cfg, args.seed, args.family, args.cpu_sample, world, inputs)
    tot, toks = 0.0, 0
    for _ in range(args.steps):
        s, n = oracle_step_sample(cfg, args.seed, args.family, args.cpu_sample, world, inputs)
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

    # N > 1: the gate weights are replicated (data parallel), so every step ends with the
    # allreduce of dWg (S8(g)) — a non-expert gradient issued through the micro-op scheduler
    # (S9) on the DP communicator; the stream waits for it on the device.
    policy = {"baseline": 0, "lina": 1, "naive": 2, "defer": 3}[args.sched_policy]
    if world > 1:
        lina.lina_sched_config(comm, policy, 30 << 20)

    def allreduce_dwg():
        if world > 1:
            lina.lina_allreduce_submit(comm, outs["dwg"], stream)
            lina.lina_allreduce_wait(comm, stream)

    def step(xx, dyy):
        layer.forward(xx, wg, w1, w2, out=outs["y"])
        layer.backward(dyy, xx, wg, w1, w2, outs["dx"], outs["dwg"], outs["dw1"], outs["dw2"])
        allreduce_dwg()

    # routing of this batch (identical every step): kept assignments for the algorithmic flop count
    layer.forward(x, wg, w1, w2, out=outs["y"], want_route=True)
    counts = layer.route_t["counts"].cpu().numpy()
    kept_local = int(np.minimum(counts, C).sum())
    progress(f"{cfg.name} N={world}: layer built, {args.warmup} warm-up steps")
    for _ in range(args.warmup):
        step(x, dy)
    torch.cuda.synchronize()
    progress("warm-up done")

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
    if graph is not None:
        def run_step():
            graph.replay()
            allreduce_dwg()  # (host-issued micro-ops: not part of the captured graph)
    else:
        def run_step():
            step(x, dy)

    progress(f"launch mode: {launch_mode}")
    # ---------------- timed region (device time, per-step events, L2 flushed between steps)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        barrier()
        torch.cuda.synchronize()
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
    progress(f"timed region done: median {np.median(step_ms):.3f} ms/step")

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
    step_ms_eager = [a.elapsed_time(b) for a, b in evs_e]
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

    # ---------------- exposed communication and H(n) (N > 1): eager passes of
    # the same steps — full (T_pass, the pipelining efficiency's windows), compute-only
    # (collectives skipped: T_rest + T_ffn, with T_ffn = the expert-GEMM phases) and
    # collectives-only (the fused transport's 2n micro-ops per pass alone: T_a2a(n)).
    # Medians over the K steps; the three kinds are interleaved step by step (full, compute-only,
    # collectives-only, full, ...) so that clock changes under the power cap hit all three alike
    # (three back-to-back blocks of K steps disagreed by more than the exposed time at C5).
    def h_of(lay, nch):
        lay.forward(x, wg, w1, w2, out=outs["y"])  # routing in `saved` for the movers-only pass
        kinds = (1, 1 | 2, 4)
        got = {f: [] for f in kinds}
        for i in range(args.steps):
            for flags in kinds:
                lina.lina_profile_enable(comm, flags)
                barrier()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                flush.zero_()
                e0.record(stream)
                lay.forward(x, wg, w1, w2, out=outs["y"])
                lay.backward(dy, x, wg, w1, w2, outs["dx"], outs["dwg"], outs["dw1"], outs["dw2"])
                e1.record(stream)
                torch.cuda.synchronize()
                lina.lina_profile_enable(comm, 0)
                pr = lina.lina_profile_read(comm)
                got[flags].append((e0.elapsed_time(e1), pr["gemm_ms"], pr["a2a_window_ms"], pr["gemm_in_a2a_ms"]))
        barrier()

        def med(flags):
            v = torch.tensor(np.median(np.array(got[flags], dtype=np.float64), axis=0), dtype=torch.float64,
                             device=dev)
            torch.distributed.all_reduce(v, op=torch.distributed.ReduceOp.MAX)
            return [float(t) for t in v]
        t_pass, _, win, busy = med(1)
        t_comp, t_ffn, _, _ = med(1 | 2)
        t_a2a = med(4)[0]
        lay.forward(x, wg, w1, w2, out=outs["y"])  # (restore real routing / rounds)
        lay.backward(dy, x, wg, w1, w2, outs["dx"], outs["dwg"], outs["dw1"], outs["dw2"])
        torch.cuda.synchronize()
        t_rest = max(0.0, t_comp - t_ffn)
        X = max(0.0, t_pass - t_comp)
        O = min(t_a2a * (1.0 - 1.0 / nch), t_ffn)  # fill (first dispatch) and drain (last combine)
        elt_ = 2 if tdt == torch.bfloat16 else 4
        a2a_bytes = 4.0 * kept_local * d * elt_ * (world - 1) / world  # algorithmic, off-GPU, per rank
        return {"n_chunks": nch, "T_pass_ms": t_pass, "T_rest_ms": t_rest, "T_ffn_ms": t_ffn,
                "T_a2a_ms": t_a2a, "exposed_ms": X,
                "overlappable_ms": O,
                "H": (min(1.0, (t_a2a - X) / O) if O > 1e-9 else None),
                "hidden_vs_isolated": max(0.0, min(1.0, 1.0 - X / t_a2a)) if t_a2a > 0 else None,
                "pipelining_efficiency": (busy / win) if win > 0 else None,
                "a2a_window_ms": win, "gemm_in_a2a_window_ms": busy,
                # nccl-tests convention: algbw = bytes each rank sends (its own experts' rows
                # included) / T_a2a; busbw = algbw (P-1)/P = the off-GPU bytes / T_a2a
                "a2a_algbw_GBps": a2a_bytes * world / (world - 1) / (t_a2a / 1e3) / 1e9 if t_a2a > 0 else None,
                "a2a_busbw_GBps": a2a_bytes / (t_a2a / 1e3) / 1e9 if t_a2a > 0 else None}

    a2a = None
    sweep = None
    if world > 1:
        progress("exposed-communication passes")
        h = h_of(layer, n_chunks)
        a2a = dict(h)
        a2a.update({
            "transport": transport,
            "definitions": "SURVEY.md §8(d): X = max(0, T_pass - T_rest - T_ffn); O = min(T_a2a(1 - 1/n), T_ffn) "
                           "(equal micro-ops: fill = first dispatch, drain = last combine); H = min(1, (T_a2a - X)/O), "
                           "null when O = 0 (n = 1: nothing overlappable under the paper's model although the fused "
                           "epilogue stores overlap the GEMM); hidden_vs_isolated = 1 - X/T_a2a; pipelining "
                           "efficiency = expert-GEMM time inside the all-to-all windows / the windows (P:700); "
                           "busbw = algorithmic off-GPU bytes (4 all-to-alls of the kept rows x (P-1)/P) / T_a2a",
            "bytes_per_rank_per_step": 4.0 * kept_local * d * (2 if tdt == torch.bfloat16 else 4) * (world - 1) / world,
            "dwg_allreduce": f"lina_allreduce_submit/wait every step, policy {args.sched_policy}, 30 MB micro-ops"})
        if args.sweep_chunks:
            sweep = []
            for nch in [int(v) for v in args.sweep_chunks.split(",") if v.strip()]:
                if nch == n_chunks:
                    sweep.append(h)
                    continue
                lay = lina.MoELayer(comm, T, d, f, E, k, C, nch, tdt, dev)
                for _ in range(2):
                    lay.forward(x, wg, w1, w2, out=outs["y"])
                    lay.backward(dy, x, wg, w1, w2, outs["dx"], outs["dwg"], outs["dw1"], outs["dw2"])
                torch.cuda.synchronize()
                progress(f"sweep n_chunks={nch}")
                sweep.append(h_of(lay, nch))
                del lay
                torch.cuda.empty_cache()

    # ---------------- end to end through the public API, host buffers (pinned), copies timed
    # Every step copies its inputs (x, dY) from pinned host memory and its results (y, dX)
    # back to pinned host memory inside the timed region.  The copies run on two copy
    # streams, double-buffered, so step i+1's inputs and step i-1's results move while
    # step i computes (the way a training input pipeline feeds the layer).
    e2e = None
    if not args.no_e2e:
        progress("end-to-end pass")
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
            allreduce_dwg()
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
    clk = clocks.summary()
    tc_peak, peak_kind, peak_why = choose_peak(pk, clk)
    elt = 2 if tdt == torch.bfloat16 else 4
    fl = gemm_floors(d, f, E // world, kept_local, elt, pk, tc_peak)
    flops_per_step_local, bytes_per_step_local = fl["flops"], fl["bytes"]
    t_tensor_ms, t_hbm_ms, hbm_bound = fl["tensor_ms"], fl["hbm_ms"], fl["hbm_bound"]
    gemm_ms_per_step = gemm_ms / max(args.steps, 1)
    if hbm_bound:
        achieved = bytes_per_step_local / (gemm_ms_per_step / 1e3) / 1e9 if gemm_ms > 0 else None
        peak, unit, psrc = pk["hbm"], "GB/s", f"{pk['src']} HBM copy bandwidth (MEASURED_PEAKS.json hbm_gbs)"
    else:
        achieved = flops_per_step_local / (gemm_ms_per_step / 1e3) / 1e12 if gemm_ms > 0 else None
        key = "bf16_tflops" if peak_kind == "burst" else "bf16_tflops_sustained"
        peak, unit, psrc = tc_peak, "TFLOP/s", f"{pk['src']} bf16 {peak_kind} (MEASURED_PEAKS.json {key}): {peak_why}"
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.config)
        except Exception:
            traffic = None
    step_med_ms = float(np.median(step_ms))
    lf = layer_floor(d, f, E // world, k, T, kept_local, world, elt, tc_peak, pk["hbm"])
    roof = {"bound": "hbm" if hbm_bound else "tensor",
            "kernel": "expert grouped GEMMs (fwd GEMM1+ReLU, GEMM2; bwd dgrad x2, wgrad x2)",
            "achieved": achieved, "peak": peak, "unit": unit,
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "peak_kind": peak_kind, "peak_src": psrc,
            "how": "achieved = algorithmic flops per step (12*k*d*f per kept assignment) / the expert-GEMM phase "
                   "time per step (CUDA events on the compute stream around every GEMM phase, eager pass)",
            "gemm_ms_per_step": gemm_ms_per_step,
            "gemm_share_of_step": gemm_ms_per_step / (sum(step_ms_eager) / args.steps) if step_ms_eager else None,
            "algorithmic_flops_per_step": flops_per_step_local,
            "algorithmic_bytes_per_step": bytes_per_step_local,
            "floors_ms": {"tensor": t_tensor_ms, "hbm": t_hbm_ms},
            # the whole layer against max(GEMM/TC, a2a/NVLink) + memory-bound/HBM
            "layer": {"t_roof_ms": lf["t_roof_ms"], "t_measured_ms": step_med_ms,
                      "frac": lf["t_roof_ms"] / step_med_ms if step_med_ms > 0 else None,
                      "terms_ms": {"gemm_tensor": lf["t_gemm_ms"], "a2a_nvlink": lf["t_a2a_ms"],
                                   "memory_bound_kernels_hbm": lf["t_mem_ms"]},
                      "bytes": {"a2a_per_direction": lf["a2a_bytes_per_direction"],
                                "memory_bound_kernels": lf["memkernel_bytes"]},
                      "peaks": {"tensor_TFLOPs": tc_peak, "hbm_GBps": pk["hbm"], "nvlink_GBps_per_direction": 900.0}}}

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
            "a2a_sweep": sweep,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(prof["kernel_launches"]),  # this library's kernels per K steps (eager count)
            "clocks": clk,
            "step_ms": {"min": min(step_ms), "median": float(np.median(step_ms)), "max": max(step_ms)},
            "host_enqueue_ms_per_step": host_ms,
        }
        print(json.dumps(line), flush=True)
    comm.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
