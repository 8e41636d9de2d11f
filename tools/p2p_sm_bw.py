"""SM-driven NVLink bandwidth probe (diagnostic): a grid-stride 16-byte copy kernel
moving a buffer local->local, local->peer (push, stores over NVLink) and peer->local
(pull, loads over NVLink), one direction and both GPUs at once.  Device-timed.
    python tools/p2p_sm_bw.py        (needs 2 GPUs; JIT-compiles a tiny extension)"""
import json

import torch
from torch.utils.cpp_extension import load_inline

SRC = r"""
#include <torch/extension.h>
#include <cuda_runtime.h>
__global__ void copy16(const uint4* __restrict__ s, uint4* __restrict__ d, long long n) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long st = (long long)gridDim.x * blockDim.x;
  for (; i + 3 * st < n; i += 4 * st) {
    uint4 a = s[i], b = s[i + st], c = s[i + 2 * st], e = s[i + 3 * st];
    d[i] = a; d[i + st] = b; d[i + 2 * st] = c; d[i + 3 * st] = e;
  }
  for (; i < n; i += st) d[i] = s[i];
}
// permute-like pattern: warp w moves R=4 rows of 1536 B (96 uint4, 3 per lane);
// rows of "expert" e = row / rows_per_e go to dst_remote when e is odd, else dst_local.
__global__ void rows4(const uint4* __restrict__ s, uint4* __restrict__ dl, uint4* __restrict__ dr, int nrows,
                      int rows_per_e) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int r0 = w * 4;
  if (r0 >= nrows) return;
  uint4 b[4][3];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) b[i][j] = s[(size_t)((r0 + i) % 8192) * 96 + lane + 32 * j];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + i;
    if (r >= nrows) break;
    uint4* d = (((r / rows_per_e) & 1) ? dr : dl) + (size_t)r * 96;
#pragma unroll
    for (int j = 0; j < 3; ++j) d[lane + 32 * j] = b[i][j];
  }
}
void rows(long long src, long long dl, long long dr, int nrows, int rows_per_e, long long stream) {
  const int warps = (nrows + 3) / 4;
  rows4<<<(warps * 32 + 255) / 256, 256, 0, (cudaStream_t)stream>>>((const uint4*)src, (uint4*)dl, (uint4*)dr,
                                                                     nrows, rows_per_e);
}
void enable_peer(int a, int b) {
  cudaSetDevice(a);
  cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
  if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) throw std::runtime_error(cudaGetErrorString(e));
  cudaGetLastError();
}
void copy(long long src, long long dst, long long bytes, int blocks, int threads, long long stream) {
  copy16<<<blocks, threads, 0, (cudaStream_t)stream>>>((const uint4*)src, (uint4*)dst, bytes / 16);
}
"""
CPP = "void rows(long long src, long long dl, long long dr, int nrows, int rows_per_e, long long stream); void enable_peer(int a, int b); void copy(long long src, long long dst, long long bytes, int blocks, int threads, long long stream);"
ext = load_inline("p2p_sm_bw", cpp_sources=CPP, cuda_sources=SRC.replace("#include <torch/extension.h>\n", ""),
                  functions=["enable_peer", "copy", "rows"], extra_cuda_cflags=["-O3"], verbose=False)
ext.enable_peer(0, 1)
ext.enable_peer(1, 0)
NB = 64 << 20
buf = {g: [torch.empty(NB, dtype=torch.uint8, device=f"cuda:{g}") for _ in range(2)] for g in (0, 1)}


def run(pairs, blocks, threads=256, reps=20):
    """pairs: list of (launch_dev, src_tensor, dst_tensor); all launched together."""
    evs = []
    for dev, s, d in pairs:
        with torch.cuda.device(dev):
            st = torch.cuda.current_stream()
            ext.copy(s.data_ptr(), d.data_ptr(), NB, blocks, threads, st.cuda_stream)  # warm
            torch.cuda.synchronize()
    for dev, s, d in pairs:
        with torch.cuda.device(dev):
            st = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(reps):
                ext.copy(s.data_ptr(), d.data_ptr(), NB, blocks, threads, st.cuda_stream)
            e1.record(st)
            evs.append((dev, e0, e1))
    out = []
    for dev, e0, e1 in evs:
        torch.cuda.synchronize(dev)
        out.append(NB * reps / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return out


for blocks in (148, 296, 592, 1184):
    r = {"blocks": blocks}
    r["local_copy"] = run([(0, buf[0][0], buf[0][1])], blocks)[0]
    r["push_0to1"] = run([(0, buf[0][0], buf[1][1])], blocks)[0]
    r["pull_1to0"] = run([(0, buf[1][0], buf[0][1])], blocks)[0]
    r["push_both"] = run([(0, buf[0][0], buf[1][1]), (1, buf[1][0], buf[0][1])], blocks)
    r["pull_both"] = run([(0, buf[1][0], buf[0][1]), (1, buf[0][0], buf[1][1])], blocks)
    print(json.dumps({k: (round(v, 1) if isinstance(v, float) else ([round(x, 1) for x in v] if isinstance(v, list) else v)) for k, v in r.items()}), flush=True)


def rows_case(both, remote=True, reps=20):
    nrows, rpe = 20480, 2560
    res = []
    devs = (0, 1) if both else (0,)
    evs = []
    for rep in range(2):
        evs = []
        for g in devs:
            o = 1 - g
            dl = buf[g][1]
            dr = buf[o][1] if remote else buf[g][0]
            with torch.cuda.device(g):
                st = torch.cuda.current_stream()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(reps if rep else 1):
                    ext.rows(xsrc[g].data_ptr(), dl.data_ptr(), dr.data_ptr(), nrows, rpe, st.cuda_stream)
                e1.record(st)
                evs.append((g, e0, e1))
        for g, e0, e1 in evs:
            torch.cuda.synchronize(g)
    return [round(e0.elapsed_time(e1) / reps * 1e3, 1) for g, e0, e1 in evs]


xsrc = {g: torch.empty(8192 * 1536, dtype=torch.uint8, device=f"cuda:{g}") for g in (0, 1)}
print(json.dumps({"rows_us_local_only": rows_case(False, remote=False), "rows_us_half_remote": rows_case(False),
                  "rows_us_half_remote_both": rows_case(True)}), flush=True)


# ---- 4-GPU all-to-all row pattern (when 4 GPUs are visible): every GPU moves 20480 rows
# of 1536 B, rows of "expert group" g (4 groups) go to GPU g (its own group stays local),
# groups visited starting at (me + 1) % 4 -- the fused permute's pattern at P = 4.
if torch.cuda.device_count() >= 4:
    G = 4
    for a_ in range(G):
        for b_ in range(G):
            if a_ != b_:
                ext.enable_peer(a_, b_)
    src4 = {g: torch.empty(8192 * 1536, dtype=torch.uint8, device=f"cuda:{g}") for g in range(G)}
    dst4 = {g: torch.empty(20480 * 1536, dtype=torch.uint8, device=f"cuda:{g}") for g in range(G)}
    SRC2 = None

    def run4(reps=20):
        evs = []
        for rep in range(2):
            evs = []
            for g in range(G):
                with torch.cuda.device(g):
                    st = torch.cuda.current_stream()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    for _ in range(reps if rep else 1):
                        for j in range(1, G + 1):  # rotated: peers first, own group last
                            o = (g + j) % G
                            # 5120 rows for owner o: local dst if o == g
                            ext.rows(src4[g].data_ptr(), dst4[o].data_ptr(), dst4[o].data_ptr(), 5120, 5120,
                                     st.cuda_stream)
                    e1.record(st)
                    evs.append((g, e0, e1))
            for g, e0, e1 in evs:
                torch.cuda.synchronize(g)
        return [round(e0.elapsed_time(e1) / reps * 1e3, 1) for g, e0, e1 in evs]

    print(json.dumps({"rows4_us_alltoall (4 x 5120 rows of 1536 B per GPU, 3/4 remote)": run4()}), flush=True)
