// S8 (e)+(f): gate backward, token gradient dX and gate-weight gradient dWg.
//
//   dL_t = p_t ∘ (dp_t − <p_t, dp_t>)                            (softmax backward, R13)
//   dX_t = Σ_{j kept} dXe[row(t,j)] + Σ_e dL_te · Wg[:, e]      (gather-sum + dL·Wgᵀ)
//   dWg  = Σ_t X_tᵀ dL_t                                         (this rank's tokens, R12)
// dp_t comes from the gate-weight gradients dg through the top-k normalisation (R4):
// k=1: g0 = p_e0 => dp_e0 = dg0; k>=2: g_j = p_ej / S => dp_ei = (dg_i − Σ_j g_j dg_j)/S;
// dp = 0 off the selected experts.  dL is a few flops per (token, expert), so it is
// recomputed inside both kernels from (probs, idx, gate, dg) instead of being a kernel
// and an HBM round trip of its own.  dX and dWg are small-K / small-N products around the
// gate (K = N = E <= 64): HBM/latency-bound, so they are register-blocked SIMT tiles
// that issue all their 16-byte loads before the first use.
//
// dx  : CTA = 32 tokens x 256 columns, thread = 4 tokens x 8 columns (one 16-byte
//       vector per token).  The Wg slab for the CTA's columns (contiguous in Wg) is
//       staged transposed ([e][col], swizzled for conflict-free float4 reads) with the
//       dL tile (8 threads per token);
//       each e step is 32 FMAs for 6 shared loads.  The expert-gradient rows are
//       gathered with one 16-byte load per (token, kept j).
// dwg : CTA = 256 columns x 4 experts x 128 tokens, thread = 8 columns x 4 experts,
//       8 token lanes (one per warp) each walking every 8th token in double-buffered
//       batches of 4, folded in shared memory in a fixed tree order; each token split
//       writes one partial, reduced afterwards in a fixed order (deterministic, no
//       float atomics).
#include <stdlib.h>

#include <algorithm>

#include "../common.h"
#include "../kernels.h"
#include "../signal.h"

namespace lina {
namespace {

constexpr int kDxTok = 32, kDxCols = 256;
constexpr int kDwgTok = 128, kDwgB = 4;  // tokens per dwg CTA; tokens per thread per batch
constexpr int kDwgE = 4;                  // experts per dwg CTA (grid z covers E)

// Wg slab column c = 8*cg + 4*h + q is kept at 128*h + 4*cg + q so that the float4 reads
// of one half by the 32 column groups of a warp are contiguous (no bank conflicts).
__device__ __forceinline__ int swz(int c) { return ((c >> 2) & 1) * 128 + (c >> 3) * 4 + (c & 3); }

// Per-token part of the gate backward (see the header): <p_t, dp_t> and dp_t at the k
// selected experts (es[j], dps[j]; es = -1 past k).  All loads of a token are issued
// together: the routing of the token, then the k selected probabilities.
template <int KM>
__device__ __forceinline__ float token_dp(const float* __restrict__ probs, const int* __restrict__ idx,
                                          const float* __restrict__ gate, const float* __restrict__ dg,
                                          int t, int k, int E, int (&es)[KM], float (&dps)[KM]) {
  float gg[KM], dd[KM], pp[KM];
#pragma unroll
  for (int j = 0; j < KM; ++j) {
    const bool v = j < k;
    es[j] = v ? idx[(size_t)t * k + j] : -1;
    gg[j] = v ? gate[(size_t)t * k + j] : 0.f;
    dd[j] = v ? dg[(size_t)t * k + j] : 0.f;
  }
#pragma unroll
  for (int j = 0; j < KM; ++j) pp[j] = es[j] >= 0 ? probs[(size_t)t * E + es[j]] : 0.f;
  if (k == 1) {
    dps[0] = dd[0];
#pragma unroll
    for (int j = 1; j < KM; ++j) dps[j] = 0.f;
    return pp[0] * dd[0];
  }
  float S = 0.f, sgd = 0.f;
#pragma unroll
  for (int j = 0; j < KM; ++j)
    if (j < k) {
      S += pp[j];
      sgd = fmaf(gg[j], dd[j], sgd);
    }
  float dot = 0.f;
#pragma unroll
  for (int j = 0; j < KM; ++j) {
    dps[j] = j < k ? (dd[j] - sgd) / S : 0.f;
    if (j < k) dot = fmaf(pp[j], dps[j], dot);
  }
  return dot;
}

// dL_te = p_te (dp_te − <p_t, dp_t>)
template <int KM>
__device__ __forceinline__ float dl_of(float pe, int e, float dot, const int (&es)[KM], const float (&dps)[KM]) {
  float dp = 0.f;
#pragma unroll
  for (int j = 0; j < KM; ++j)
    if (es[j] == e) dp = dps[j];
  return pe * (dp - dot);
}

template <typename T, int KT>  // KT = k when 1 or 2, 0 = generic k <= 8
__global__ void __launch_bounds__(256) dx_tiled_kernel(const T* __restrict__ dXe, const int* __restrict__ idx,
                                                       const int* __restrict__ slot,
                                                       const float* __restrict__ probs,
                                                       const float* __restrict__ gate,
                                                       const float* __restrict__ dg,
                                                       const float* __restrict__ Wg, int Tn, int k, int d,
                                                       int E, int C, int n, int Cm, T* __restrict__ dX,
                                                       PeerSignal sig, const int* __restrict__ ebase) {
  pdl_enter();
  extern __shared__ float dsm[];
  if (threadIdx.x == 0) sig_wait(sig);  // fused transport: the expert input-gradients have landed
  __syncthreads();
  float* sW = dsm;                     // [E][kDxCols]
  float* sL = dsm + E * kDxCols;       // [kDxTok][E]
  constexpr int NV = sizeof(T) == 2 ? 1 : 2;  // 16-byte vectors per 8 columns
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * kDxCols;
  const int t0 = blockIdx.y * kDxTok;
  const int cg = tid & 31, tg = tid >> 5;  // 32 column groups x 8 token groups
  const int col = c0 + cg * 8;
  // gather-sum of the returned expert input-gradients: all (slot, idx) pairs of the
  // thread's 4 tokens first, then every 16-byte row load, so they are all in flight
  constexpr int KM = KT > 0 ? KT : 8;
  int sl[4][KM], ex[4][KM];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = t0 + tg * 4 + i;
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      const bool ok = t < Tn && j < k && col < d;
      sl[i][j] = ok ? slot[(size_t)t * k + j] : -1;
      ex[i][j] = ok ? idx[(size_t)t * k + j] : 0;
    }
  }
  uint4 raw[4][KM][NV];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      const uint4* src = reinterpret_cast<const uint4*>(
          dXe + (ebase ? (size_t)(ebase[ex[i][j]] + (sl[i][j] < 0 ? 0 : sl[i][j]))   // dropless: compact rows
                       : send_row(ex[i][j], sl[i][j] < 0 ? 0 : sl[i][j], E, C, n, Cm)) * d + col);
#pragma unroll
      for (int v = 0; v < NV; ++v) raw[i][j][v] = sl[i][j] >= 0 ? src[v] : make_uint4(0, 0, 0, 0);
    }
  // Wg rows c0 .. c0+255 are contiguous ([d][E] row-major): float4 reads, transposed stores
  const int ncol = min(kDxCols, d - c0);
  if ((E & 3) == 0) {
    const float4* w4 = reinterpret_cast<const float4*>(Wg + (size_t)c0 * E);
    const int nv = ncol * E / 4;
#pragma unroll 4
    for (int i = tid; i < nv; i += 256) {
      const float4 w = __ldg(w4 + i);
      const int f = 4 * i, c = f / E, e = f % E;
      const int sc = swz(c);
      sW[(e + 0) * kDxCols + sc] = w.x;
      sW[(e + 1) * kDxCols + sc] = w.y;
      sW[(e + 2) * kDxCols + sc] = w.z;
      sW[(e + 3) * kDxCols + sc] = w.w;
    }
  } else {
    for (int i = tid; i < ncol * E; i += 256) sW[(i % E) * kDxCols + swz(i / E)] = __ldg(Wg + (size_t)c0 * E + i);
  }
  {  // dL tile: 8 threads per token, expert e = sub + 8m
    const int r = tid >> 3, sub = tid & 7, t = t0 + r;
    if (t < Tn) {
      float pe[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) pe[m] = sub + 8 * m < E ? probs[(size_t)t * E + sub + 8 * m] : 0.f;
      int es[KM];
      float dps[KM];
      const float dot = token_dp<KM>(probs, idx, gate, dg, t, k, E, es, dps);
#pragma unroll
      for (int m = 0; m < 8; ++m)
        if (sub + 8 * m < E) sL[r * E + sub + 8 * m] = dl_of<KM>(pe[m], sub + 8 * m, dot, es, dps);
    } else {
      for (int e = sub; e < E; e += 8) sL[r * E + e] = 0.f;
    }
  }
  __syncthreads();
  if (col < d) {
    float acc[4][8];
  #pragma unroll
    for (int i = 0; i < 4; ++i) {
  #pragma unroll
      for (int c = 0; c < 8; ++c) acc[i][c] = 0.f;
  #pragma unroll
      for (int j = 0; j < KM; ++j) {
        float x[8];
        if constexpr (sizeof(T) == 2) {
          load16(&raw[i][j][0], x, (const __nv_bfloat16*)nullptr);
        } else {
          load16(&raw[i][j][0], x, (const float*)nullptr);
          load16(&raw[i][j][NV - 1], x + 4, (const float*)nullptr);
        }
  #pragma unroll
        for (int c = 0; c < 8; ++c) acc[i][c] += x[c];
      }
    }
    // + dL · Wgᵀ
    for (int e = 0; e < E; ++e) {
      const float4 w0 = *reinterpret_cast<const float4*>(sW + e * kDxCols + cg * 4);
      const float4 w1 = *reinterpret_cast<const float4*>(sW + e * kDxCols + 128 + cg * 4);
      const float w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
  #pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float l = sL[(tg * 4 + i) * E + e];
  #pragma unroll
        for (int c = 0; c < 8; ++c) acc[i][c] = fmaf(l, w[c], acc[i][c]);
      }
    }
  #pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int t = t0 + tg * 4 + i;
      if (t >= Tn) continue;
      T* dst = dX + (size_t)t * d + col;
      if constexpr (sizeof(T) == 2) {
        store16(dst, acc[i], (__nv_bfloat16*)nullptr);
      } else {
        store16(dst, acc[i], (float*)nullptr);
        store16(dst + 4, acc[i] + 4, (float*)nullptr);
      }
    }
  }
  if (sig.bump) {  // the backward's last kernel closes its round
    __syncthreads();
    if (tid == 0) sig_bump_last(sig);
  }
}

// part[split][col][e] over tokens t in [split*kDwgTok, +kDwgTok): token lane l (= warp)
// takes t = ta + l + 8*i, combined over the 8 lanes in shared memory in a fixed order.
template <typename T>
__global__ void __launch_bounds__(256, 3) dwg_tiled_kernel(const T* __restrict__ X,
                                                           const float* __restrict__ probs,
                                                           const int* __restrict__ idx,
                                                           const float* __restrict__ gate,
                                                           const float* __restrict__ dg, int Tn, int d,
                                                           int E, int k, float* __restrict__ part) {
  pdl_enter();
  constexpr int EG = kDwgE;  // experts per CTA (blockIdx.z = expert group)
  __shared__ float red[4][256 * EG];
  __shared__ __align__(16) float sL[kDwgTok][EG];
  constexpr int NV = sizeof(T) == 2 ? 1 : 2;
  constexpr int NB = kDwgTok / 8 / kDwgB;  // batches per thread
  const int tid = threadIdx.x;
  const int cg = tid & 31, lane_t = tid >> 5;
  const int col = blockIdx.x * 256 + cg * 8;
  const int split = blockIdx.y;
  const int e0 = blockIdx.z * EG;
  const int ne = min(EG, E - e0);
  const int ta = split * kDwgTok;
  const bool cin = col < d;
  uint4 cur[kDwgB][NV], nxt[kDwgB][NV];
  auto load_batch = [&](int b, uint4 (&r)[kDwgB][NV]) {
#pragma unroll
    for (int i = 0; i < kDwgB; ++i) {
      const int t = ta + lane_t + 8 * (b * kDwgB + i);
      const uint4* src = reinterpret_cast<const uint4*>(X + (size_t)(t < Tn ? t : 0) * d + (cin ? col : 0));
#pragma unroll
      for (int v = 0; v < NV; ++v) r[i][v] = (cin && t < Tn) ? src[v] : make_uint4(0, 0, 0, 0);
    }
  };
  load_batch(0, cur);
  {  // dL tile: 2 threads per token, half of the CTA's EG experts each
    constexpr int EH = EG / 2;
    const int r = tid >> 1, q0 = (tid & 1) * EH, t = ta + r;
    float pe[EH];
#pragma unroll
    for (int q = 0; q < EH; ++q) pe[q] = (t < Tn && q0 + q < ne) ? probs[(size_t)t * E + e0 + q0 + q] : 0.f;
    if (t < Tn) {
      int es[8];
      float dps[8];
      const float dot = token_dp<8>(probs, idx, gate, dg, t, k, E, es, dps);
#pragma unroll
      for (int q = 0; q < EH; ++q) sL[r][q0 + q] = q0 + q < ne ? dl_of<8>(pe[q], e0 + q0 + q, dot, es, dps) : 0.f;
    } else {
#pragma unroll
      for (int q = 0; q < EH; ++q) sL[r][q0 + q] = 0.f;
    }
  }
  __syncthreads();
  float acc[8][EG];
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int q = 0; q < EG; ++q) acc[c][q] = 0.f;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (b + 1 < NB) load_batch(b + 1, (b & 1) ? cur : nxt);
    uint4 (&r)[kDwgB][NV] = (b & 1) ? nxt : cur;
#pragma unroll
    for (int i = 0; i < kDwgB; ++i) {
      float x[8];
      if constexpr (sizeof(T) == 2) {
        load16(&r[i][0], x, (const __nv_bfloat16*)nullptr);
      } else {
        load16(&r[i][0], x, (const float*)nullptr);
        load16(&r[i][NV - 1], x + 4, (const float*)nullptr);
      }
      const int tr = lane_t + 8 * (b * kDwgB + i);
      float l[EG];
#pragma unroll
      for (int q = 0; q < EG; q += 4) {
        const float4 lv = *reinterpret_cast<const float4*>(&sL[tr][q]);
        l[q] = lv.x;
        l[q + 1] = lv.y;
        l[q + 2] = lv.z;
        l[q + 3] = lv.w;
      }
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int q = 0; q < EG; ++q) acc[c][q] = fmaf(x[c], l[q], acc[c][q]);
    }
  }
  // fixed-order tree over the 8 token lanes: (0+4,1+5,2+6,3+7), (0+2,1+3), (0+1)
  for (int half = 4; half >= 1; half >>= 1) {
    if (lane_t >= half && lane_t < 2 * half) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int q = 0; q < EG; ++q) red[lane_t - half][(c * EG + q) * 32 + cg] = acc[c][q];
    }
    __syncthreads();
    if (lane_t < half) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int q = 0; q < EG; ++q) acc[c][q] += red[lane_t][(c * EG + q) * 32 + cg];
    }
    __syncthreads();
  }
  if (lane_t == 0 && cin) {
    float* dst = part + ((size_t)split * d + col) * E + e0;
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int q = 0; q < EG; ++q)
        if (q < ne) dst[(size_t)c * E + q] = acc[c][q];
  }
}

// dWg[i] = Σ_split part[split][i] in split order: CTA = 32 outputs x 8 split groups
// (consecutive split ranges, all loads in flight), groups combined in order.
constexpr int kRedG = 8;
__global__ void __launch_bounds__(256) dwg_reduce_kernel(const float* __restrict__ part, int nparts, int dE,
                                                         float* __restrict__ dWg) {
  pdl_enter();
  __shared__ float gs[kRedG][32];
  const int lane = threadIdx.x & 31, gq = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  const int per = (nparts + kRedG - 1) / kRedG;
  const int qa = gq * per, qb = min(nparts, qa + per);
  float s = 0.f;
  if (i < dE) {
    int q = qa;
    for (; q + 8 <= qb; q += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(part + (size_t)(q + u) * dE + i);
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; q < qb; ++q) s += __ldg(part + (size_t)q * dE + i);
  }
  gs[gq][lane] = s;
  __syncthreads();
  if (gq == 0 && i < dE) {
    float r = gs[0][lane];
#pragma unroll
    for (int g = 1; g < kRedG; ++g) r += gs[g][lane];
    dWg[i] = r;
  }
}

int dwg_splits(int T) { return (T + kDwgTok - 1) / kDwgTok; }

}  // namespace

size_t dwg_scratch_floats(int T, int d, int E) {
  // (also the tensor-core path's dL split and partials, gate_bwd_tc.cu)
  return std::max((size_t)dwg_splits(T) * d * E, (gate_bwd_tc_scratch_bytes(T, d, E) + 3) / 4);
}

void launch_dwg_reduce(const float* part, int nparts, int dE, float* dWg, cudaStream_t s) {
  launch_k(dwg_reduce_kernel, dim3((dE + 31) / 32), dim3(256), 0, s, part, nparts, dE, dWg);
  LINA_LAUNCH_CHECK();
}

// LINA_GATE_BWD_SIMT=1 keeps the CUDA-core dX / dWg (A/B comparisons)
static bool gate_bwd_tc_on(int dtype, int d, int E, int k) {
  static const bool simt = [] {
    const char* e = getenv("LINA_GATE_BWD_SIMT");
    return e && e[0] == '1';
  }();
  return !simt && gate_bwd_tc_supported(dtype, d, E, k);
}

template <typename T, int KT>
static void launch_dx_t(const void* dXe, const int* idx, const int* slot, const float* probs,
                        const float* gate, const float* dg, const float* Wg, int Tn, int k, int d, int E,
                        int C, int n, int Cm, void* dX, const PeerSignal& sig, cudaStream_t s,
                        const int* ebase) {
  dim3 grid((d + kDxCols - 1) / kDxCols, std::max(1, (Tn + kDxTok - 1) / kDxTok));
  const size_t smem = sizeof(float) * ((size_t)E * kDxCols + kDxTok * E);
  static bool set = false;
  if (!set) {
    LINA_CUDA_CHECK(cudaFuncSetAttribute(dx_tiled_kernel<T, KT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    set = true;
  }
  launch_k(dx_tiled_kernel<T, KT>, grid, dim3(256), smem, s, (const T*)dXe, idx, slot, probs, gate, dg, Wg, Tn, k, d,
           E, C, n, Cm, (T*)dX, sig, ebase);
}

void launch_dx(int dtype, const void* dXe, const int* idx, const int* slot, const float* probs,
               const float* gate, const float* dg, const float* Wg, int T, int k, int d, int E, int C,
               int n, int Cm, void* dX, cudaStream_t s, const PeerSignal* sig, const int* ebase,
               const void* tc_scratch) {
  if (T <= 0 && !sig) return;  // (with a signal, one CTA still closes the round)
  const PeerSignal sg = sig ? *sig : PeerSignal{};
  if (tc_scratch && gate_bwd_tc_on(dtype, d, E, k)) {  // dL split by the preceding launch_dwg
    launch_dx_tc(dXe, idx, slot, Wg, T, k, d, E, C, n, Cm, ebase, dX, tc_scratch, sg, s);
    return;
  }
  auto go = [&](auto tag) {
    using ET = decltype(tag);
    if (k == 1) launch_dx_t<ET, 1>(dXe, idx, slot, probs, gate, dg, Wg, T, k, d, E, C, n, Cm, dX, sg, s, ebase);
    else if (k == 2) launch_dx_t<ET, 2>(dXe, idx, slot, probs, gate, dg, Wg, T, k, d, E, C, n, Cm, dX, sg, s, ebase);
    else launch_dx_t<ET, 0>(dXe, idx, slot, probs, gate, dg, Wg, T, k, d, E, C, n, Cm, dX, sg, s, ebase);
  };
  if (dtype == 0) go(float{});
  else go(__nv_bfloat16{});
  LINA_LAUNCH_CHECK();
}

void launch_dwg(int dtype, const void* X, const float* probs, const int* idx, const float* gate,
                const float* dg, int T, int d, int E, int k, float* scratch, float* dWg, cudaStream_t s) {
  if (T <= 0) {
    LINA_CUDA_CHECK(cudaMemsetAsync(dWg, 0, sizeof(float) * (size_t)d * E, s));
    return;
  }
  if (gate_bwd_tc_on(dtype, d, E, k)) {
    launch_dwg_tc(X, probs, idx, gate, dg, T, d, E, k, scratch, dWg, s);
    return;
  }
  const int nsplit = dwg_splits(T);
  dim3 grid((d + 255) / 256, nsplit, (E + kDwgE - 1) / kDwgE);
  if (dtype == 0)
    launch_k(dwg_tiled_kernel<float>, grid, dim3(256), 0, s, (const float*)X, probs, idx, gate, dg, T, d, E, k,
             scratch);
  else
    launch_k(dwg_tiled_kernel<__nv_bfloat16>, grid, dim3(256), 0, s, (const __nv_bfloat16*)X, probs, idx, gate, dg,
             T, d, E, k, scratch);
  LINA_LAUNCH_CHECK();
  const int dE = d * E;
  launch_k(dwg_reduce_kernel, dim3((dE + 31) / 32), dim3(256), 0, s, scratch, nsplit, dE, dWg);
  LINA_LAUNCH_CHECK();
}

}  // namespace lina
