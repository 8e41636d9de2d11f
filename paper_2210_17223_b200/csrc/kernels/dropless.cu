// Dropless training layout: the unequal-split all-to-all of
// P:525 ("the transfer size to each device ... does not need to be the same") applied
// to training, so no capacity bound drops tokens and no buffer is sized by E·T rows.
//
// After the gate, every rank stores its per-expert counts into every peer (one 1-CTA
// kernel: the count exchange) and, from the full count table allc[P][E], every rank
// computes the same layout (one 1-CTA kernel):
//   - receive side, owner o: its experts' rows in expert-major blocks (el, s) — the rows
//     source s routes to local expert el — each block cut into "virtual segments" of R
//     rows (R = the tensor-core tile height), so the expert GEMMs run unchanged over
//     V fixed-pitch segments [V][R][w], each at most one M tile, whose weight index is
//     a per-segment table (vexp) and whose wgrad ranges are per expert (vrange);
//   - source side, rank s: its kept rows compact in (expert, slot) order, soff[s][e] =
//     Σ_{e' < e} allc[s][e'] (the returned outputs and input-gradients land there).
// Footprint: V·R <= P·T·min(k, E_l) + P·E_l·R rows per receive buffer instead of the
// padded P·E_l·T (C = T), and T·k rows per source buffer instead of E·T.
//
// Row movers (one warp per row, 16-byte vectors):
//   dl_permute     : X[t] -> owner's R at dbase[e] + slot (NVLink peer stores at P > 1)
//   dl_combine_bwd : dg[t,j] = <dY_t, O[ebase[e] + slot]>,  owner's dO row = g·dY_t
//   dl_push_vsegs  : segment rows (O or dXe) -> source s's buffer at soff[s][e] + q0
// plus zero rows [c, roundup64(c)) after every (el, s) block: the wgrad reads rows in
// 64-row K blocks (the same padding rule as the capacity layout).
#include <cuda_bf16.h>

#include <algorithm>

#include "../common.h"
#include "../kernels.h"

namespace lina {
namespace {

// 1 CTA: wait for the peers' FREE, store this rank's kept[E] into row `me` of every
// rank's count table (its own included), publish READY of the counts.
__global__ void dl_counts_kernel(const int* __restrict__ kept, int* const* __restrict__ peer_allc, int P, int me,
                                 int E, PeerSignal sig) {
  pdl_enter();
  if (threadIdx.x == 0) sig_wait(sig);
  __syncthreads();
  for (int i = threadIdx.x; i < P * E; i += blockDim.x) {
    const int o = (i / E + me + 1) % P;  // every rank starts with a different owner
    peer_allc[o][me * E + i % E] = kept[i % E];
  }
  __syncthreads();
  if (threadIdx.x == 0) sig_post(sig);  // (sig_post fences system-wide before publishing)
}

// 1 CTA (256 threads): the layout tables from allc [P][E].  kMaxPE = P·E <= 8·64.
// Expert packing m (pack): rank o hosts the El = m·E/P experts of group o / m and receives
// from the Q = P/m sources s with s % m == o % m; its blocks are (el, j), j = s / m, so
// every owner has El·Q = E blocks.
constexpr int kMaxPE = 512;
__global__ void __launch_bounds__(256) dl_layout_kernel(const int* __restrict__ allc, int P, int E, int El, int m,
                                                        int me, int R, int V, int split, DlTables t) {
  pdl_enter();
  __shared__ int cnt[kMaxPE];
  __shared__ int vb[kMaxPE];     // [o][el][j]: first virtual segment of block (el, j) at owner o
  __shared__ int soff[kMaxPE];   // [s][e]: compact source offsets
  __shared__ int used[8];        // segments used per owner
  const int Q = P / m;
  for (int i = threadIdx.x; i < P * E; i += blockDim.x) cnt[i] = allc[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int w = warp; w < 2 * P; w += blockDim.x >> 5) {
    if (w < P) {  // owner o = w: exclusive prefix over its blocks (el, j) of ceil(count / R)
      const int o = w;
      int run = 0;
      for (int b = 0; b < E; b += 32) {
        const int i = b + lane;
        int v = 0;
        if (i < E) {
          const int el = i / Q, s = (i % Q) * m + o % m;
          v = (cnt[s * E + (o / m) * El + el] + R - 1) / R;
        }
        int x = v;  // inclusive warp scan
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, dd);
          if (lane >= dd) x += y;
        }
        if (i < E) vb[o * E + i] = run + x - v;
        run += __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) used[o] = run;
    } else {  // source s = w - P: exclusive prefix over e of its counts
      const int s = w - P;
      int run = 0;
      for (int b = 0; b < E; b += 32) {
        const int e = b + lane;
        const int v = e < E ? cnt[s * E + e] : 0;
        int x = v;
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, dd);
          if (lane >= dd) x += y;
        }
        if (e < E) soff[s * E + e] = run + x - v;
        run += __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) t.src_total[s] = run;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < P * E; i += blockDim.x) t.soff[i] = soff[i];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int o = (e / El) * m + me % m, el = e % El;  // the group member that takes my rows of e
    t.dbase[e] = vb[o * E + el * Q + me / m] * R;
    t.ebase[e] = P > 1 ? soff[me * E + e] : vb[el] * R;  // (P = 1: m = Q = 1, o = 0)
  }
  const int U = used[me];
  // this rank's segments: block (el, j) -> ceil(c / R) segments of R rows
  for (int i = threadIdx.x; i < E; i += blockDim.x) {
    const int el = i / Q, s = (i % Q) * m + me % m;
    const int c = cnt[s * E + (me / m) * El + el];
    const int b = vb[me * E + i];
    for (int j = 0; j * R < c; ++j) {
      t.vcount[b + j] = min(R, c - j * R);
      t.vexp[b + j] = el;
      t.vsrc[b + j] = s;
      t.vq0[b + j] = j * R;
    }
  }
  for (int v = U + threadIdx.x; v < V; v += blockDim.x) {
    t.vcount[v] = 0;
    t.vexp[v] = 0;
    t.vsrc[v] = 0;
    t.vq0[v] = 0;
  }
  if (!split) {
    for (int v = threadIdx.x; v <= V; v += blockDim.x) t.mtp[v] = min(v, U);  // one M tile per used segment
  } else {  // tail split: segments of > 128 rows as 256-row tiles, the others as 128-row tiles
    __syncthreads();  // (the vcount stores above are visible to the block after this)
    if (threadIdx.x == 0) {
      int a = 0, b = 0;
      for (int v = 0; v < V; ++v) {
        t.mtp[v] = a;
        t.mtpt[v] = b;
        const int c = t.vcount[v];
        a += c > 128 ? 1 : 0;
        b += (c > 0 && c <= 128) ? 1 : 0;
      }
      t.mtp[V] = a;
      t.mtpt[V] = b;
    }
  }
  for (int el = threadIdx.x; el < El; el += blockDim.x) {
    t.vrange[2 * el] = vb[me * E + el * Q];
    t.vrange[2 * el + 1] = el + 1 < El ? vb[me * E + (el + 1) * Q] : U;
  }
}

// Expert of compact source row r (binary search over this rank's E + 1 offsets).
__device__ __forceinline__ int expert_of_row(const int* __restrict__ off, int E, int total, int r) {
  int lo = 0, hi = E - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= r) lo = mid;
    else hi = mid - 1;
  }
  (void)total;
  return lo;
}

// Data items: compact rows [0, total); pad items: E x 64 (rows [c_e, roundup64(c_e)) of every block).
template <bool BWD>
__global__ void __launch_bounds__(256) dl_rows_kernel(const uint4* __restrict__ X, const int* __restrict__ tok_of,
                                                      const int* __restrict__ kept, const int* __restrict__ soff_me,
                                                      const int* __restrict__ dbase, const int* __restrict__ total_p,
                                                      int C, int k, int E, int El, int m, int me, int nv,
                                                      uint4* const* __restrict__ dst,
                                                      uint4* __restrict__ dst_local,  // when dst == NULL
                                                      // BWD: dY = X, rows of O at ebase, gate, dg out
                                                      const uint4* __restrict__ O, const int* __restrict__ ebase,
                                                      const float* __restrict__ gate, float* __restrict__ dg,
                                                      PeerSignal sig, int rot_expert) {
  pdl_enter();
  __shared__ int off[65];
  for (int e = threadIdx.x; e < E; e += blockDim.x) off[e] = soff_me[e];
  if (sig.wait) {
    if (threadIdx.x == 0) sig_wait(sig);
  }
  __syncthreads();
  // peer stores: every rank starts with the rows of owner (me + 1) % P (its first expert
  // rot_expert), so at any moment the ranks write to different owners (no incast)
  const int rot = rot_expert >= 0 ? off[rot_expert] : 0;
  const int total = *total_p;  // this rank's kept rows (T·k when nothing is dropped)
  const int lane = threadIdx.x & 31;
  const long long items = (long long)total + (long long)E * 64;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < items; w += nw) {
    long long it = w;
    if (it < total) {
      // rotate the data rows so the ranks start with different owners (no incast)
      it += rot;
      if (it >= total) it -= total;
      const int r = (int)it;
      const int e = expert_of_row(off, E, total, r);
      const int q = r - off[e];
      const int a = tok_of[(size_t)e * C + q];  // (tok_of pitch: the capacity C)
      const int t = a / k;
      uint4* to = (dst ? dst[(e / El) * m + me % m] : dst_local) + (size_t)(dbase[e] + q) * nv;
      const uint4* xr = X + (size_t)t * nv;
      if constexpr (!BWD) {
        for (int v = lane; v < nv; v += 32) to[v] = xr[v];
      } else {
        const uint4* orow = O + (size_t)(ebase[e] + q) * nv;
        const float g = gate[a];
        float dot = 0.f;
        for (int v = lane; v < nv; v += 32) {
          const uint4 y = xr[v], o = orow[v];
          const __nv_bfloat162* yh = reinterpret_cast<const __nv_bfloat162*>(&y);
          const __nv_bfloat162* oh = reinterpret_cast<const __nv_bfloat162*>(&o);
          uint4 outv;
          __nv_bfloat162* wh = reinterpret_cast<__nv_bfloat162*>(&outv);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float2 yf = __bfloat1622float2(yh[u]), of = __bfloat1622float2(oh[u]);
            dot = fmaf(yf.x, of.x, dot);
            dot = fmaf(yf.y, of.y, dot);
            wh[u] = __floats2bfloat162_rn(g * yf.x, g * yf.y);
          }
          to[v] = outv;
        }
#pragma unroll
        for (int dd = 16; dd > 0; dd >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, dd);
        if (lane == 0) dg[a] = dot;
      }
    } else {
      const long long p = it - total;
      const int e = (int)(p / 64), i = (int)(p % 64);
      const int c = kept[e], q = c + i;
      if (q >= ((c + 63) & ~63)) continue;
      uint4* to = (dst ? dst[(e / El) * m + me % m] : dst_local) + (size_t)(dbase[e] + q) * nv;
      for (int v = lane; v < nv; v += 32) to[v] = make_uint4(0, 0, 0, 0);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) sig_post_last(sig);
}

// fp32 backward rows (the CUDA-core path at P = 1)
__global__ void __launch_bounds__(256) dl_combine_bwd_f32_kernel(const float4* __restrict__ dY,
                                                                 const int* __restrict__ tok_of,
                                                                 const int* __restrict__ kept,
                                                                 const int* __restrict__ soff_me,
                                                                 const int* __restrict__ dbase,
                                                                 const int* __restrict__ total_p, int C,
                                                                 int k, int E, int nv, float4* __restrict__ dO,
                                                                 const float4* __restrict__ O,
                                                                 const int* __restrict__ ebase,
                                                                 const float* __restrict__ gate,
                                                                 float* __restrict__ dg) {
  pdl_enter();
  __shared__ int off[65];
  for (int e = threadIdx.x; e < E; e += blockDim.x) off[e] = soff_me[e];
  __syncthreads();
  const int total = *total_p;
  const int lane = threadIdx.x & 31;
  const long long items = (long long)total + (long long)E * 64;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < items; w += nw) {
    if (w < total) {
      const int r = (int)w;
      const int e = expert_of_row(off, E, total, r);
      const int q = r - off[e];
      const int a = tok_of[(size_t)e * C + q];  // (tok_of pitch: the capacity C)
      const float4* yr = dY + (size_t)(a / k) * nv;
      const float4* orow = O + (size_t)(ebase[e] + q) * nv;
      float4* to = dO + (size_t)(dbase[e] + q) * nv;
      const float g = gate[a];
      float dot = 0.f;
      for (int v = lane; v < nv; v += 32) {
        const float4 y = yr[v], o = orow[v];
        dot = fmaf(y.x, o.x, dot);
        dot = fmaf(y.y, o.y, dot);
        dot = fmaf(y.z, o.z, dot);
        dot = fmaf(y.w, o.w, dot);
        to[v] = make_float4(g * y.x, g * y.y, g * y.z, g * y.w);
      }
#pragma unroll
      for (int dd = 16; dd > 0; dd >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, dd);
      if (lane == 0) dg[a] = dot;
    } else {
      const long long p = w - total;
      const int e = (int)(p / 64), i = (int)(p % 64);
      const int c = kept[e], q = c + i;
      if (q >= ((c + 63) & ~63)) continue;
      float4* to = dO + (size_t)(dbase[e] + q) * nv;
      for (int v = lane; v < nv; v += 32) to[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

// grid (x, V): the valid rows of segment v to source vsrc[v] at soff[s][me*El + el] + q0.
__global__ void __launch_bounds__(256) dl_push_vsegs_kernel(const uint4* __restrict__ src,
                                                            uint4* const* __restrict__ peer, DlTables t, int R,
                                                            int E, int El, int m, int me, int nv, PeerSignal sig) {
  pdl_enter();
  const int v = blockIdx.y;
  const int rows = t.vcount[v];
  if (rows > 0) {
    const int s = t.vsrc[v], e = (me / m) * El + t.vexp[v];  // (my group's expert)
    const uint4* from = src + (size_t)v * R * nv;
    uint4* to = peer[s] + (size_t)(t.soff[s * E + e] + t.vq0[v]) * nv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int r = blockIdx.x * 8 + warp; r < rows; r += gridDim.x * 8)
      for (int u = lane; u < nv; u += 32) to[(size_t)r * nv + u] = from[(size_t)r * nv + u];
  }
  __syncthreads();
  if (threadIdx.x == 0) sig_post_last(sig);
}

// first expert whose rows go to rank (me + 1) % P: the group of that rank (packing m)
int rot_expert(void* const* peer, int me, int P, int El, int m) {
  if (!peer || P <= 1) return -1;
  const int o = (me + 1) % P;
  return (o % m == me % m) ? (o / m) * El : ((me / m + 1) % (P / m)) * El;
}

int row_blocks(long long items) {
  const long long warps = std::max(1LL, items);
  return (int)std::min<long long>(148LL * 8, (warps + 7) / 8);
}

}  // namespace

void launch_dl_counts(const int* kept, int* const* peer_allc, int P, int me, int E, const PeerSignal& sig,
                      cudaStream_t s) {
  launch_k(dl_counts_kernel, dim3(1), dim3(256), 0, s, kept, peer_allc, P, me, E, sig);
  LINA_LAUNCH_CHECK();
}

void launch_dl_layout(const int* allc, int P, int E, int El, int m, int me, int R, int V, int split, const DlTables& t,
                      cudaStream_t s) {
  if (P * E > kMaxPE || P > 8) throw CudaError{"dropless layout: P*E > 512 or P > 8"};
  launch_k(dl_layout_kernel, dim3(1), dim3(256), 0, s, allc, P, E, El, m, me, R, V, split, t);
  LINA_LAUNCH_CHECK();
}

void launch_dl_permute(int dtype, const void* X, const int* tok_of, const int* kept, const DlTables& t, int me,
                       int T, int C, int k, int E, int El, int m, int d, void* const* peer_dst, void* local_dst,
                       const PeerSignal& sig, cudaStream_t s) {
  const int elt = dtype == 1 ? 2 : 4;
  const int P = E / El * m;
  launch_k(dl_rows_kernel<false>, dim3(row_blocks((long long)T * k + 64LL * E)), dim3(256), 0, s, (const uint4*)X,
           tok_of, kept, t.soff + (size_t)me * E, t.dbase, t.src_total + me, C, k, E, El, m, me, d * elt / 16,
           (uint4* const*)peer_dst, (uint4*)local_dst, (const uint4*)nullptr, (const int*)nullptr,
           (const float*)nullptr, (float*)nullptr, sig, rot_expert(peer_dst, me, P, El, m));
  LINA_LAUNCH_CHECK();
}

void launch_dl_combine_bwd(int dtype, const void* dY, const void* O, const int* tok_of, const int* kept,
                           const float* gate, const DlTables& t, int me, int T, int C, int k, int E, int El, int m, int d,
                           void* const* peer_dst, void* local_dst, float* dg, const PeerSignal& sig, cudaStream_t s) {
  const int P = E / El * m;
  const dim3 grid(row_blocks((long long)T * k + 64LL * E));
  if (dtype == 1) {
    launch_k(dl_rows_kernel<true>, grid, dim3(256), 0, s, (const uint4*)dY, tok_of, kept, t.soff + (size_t)me * E,
             t.dbase, t.src_total + me, C, k, E, El, m, me, d * 2 / 16, (uint4* const*)peer_dst, (uint4*)local_dst,
             (const uint4*)O, t.ebase, gate, dg, sig, rot_expert(peer_dst, me, P, El, m));
  } else {
    if (peer_dst) throw CudaError{"dropless fp32 path is single-GPU"};
    launch_k(dl_combine_bwd_f32_kernel, grid, dim3(256), 0, s, (const float4*)dY, tok_of, kept,
             t.soff + (size_t)me * E, t.dbase, t.src_total + me, C, k, E, d / 4, (float4*)local_dst,
             (const float4*)O, t.ebase, gate, dg);
  }
  LINA_LAUNCH_CHECK();
}

void launch_dl_push_vsegs(int dtype, const void* src, void* const* peer, const DlTables& t, int V, int R, int E,
                          int El, int m, int me, int d, const PeerSignal& sig, cudaStream_t s) {
  const int elt = dtype == 1 ? 2 : 4;
  dim3 grid(std::max(1, std::min(8, R / 32)), std::max(1, V));
  launch_k(dl_push_vsegs_kernel, grid, dim3(256), 0, s, (const uint4*)src, (uint4* const*)peer, t, R, E, El, m, me,
           d * elt / 16, sig);
  LINA_LAUNCH_CHECK();
}

}  // namespace lina
