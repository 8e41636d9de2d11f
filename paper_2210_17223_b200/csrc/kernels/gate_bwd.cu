// S8 (e)+(f): token gradient dX and gate-weight gradient dWg.
//
//   dX_t = Σ_{j kept} dXe[row(t,j)] + Σ_e dL_te · Wg[:, e]      (gather-sum + dL·Wgᵀ)
//   dWg  = Σ_t X_tᵀ dL_t                                         (this rank's tokens, R12)
// with dL from gate_bwd_kernel (permute.cu).  Both are small-K / small-N products
// around the gate (K = N = E <= 64): they are HBM/latency-bound, so instead of a
// tensor-core tile they are register-blocked SIMT tiles that keep many 16-byte
// loads in flight.
//
// dx  : CTA = 32 tokens x 256 columns, thread = 4 tokens x 8 columns (one 16-byte
//       vector per token).  The Wg slab for the CTA's columns is staged transposed
//       ([e][col], conflict-free float4 reads) with the dL tile; each e step is 32
//       FMAs for 6 shared loads.  The expert-gradient rows are gathered with one
//       16-byte load per (token, kept j).
// dwg : CTA = 256 columns x 8 experts over a token range, thread = 8 columns x 8
//       experts, 8 token lanes (one per warp) each walking every 8th token, folded
//       in shared memory in a fixed tree order; each split writes one partial,
//       reduced afterwards in a fixed order (deterministic, no float atomics).
#include "../common.h"
#include "../kernels.h"

namespace lina {
namespace {

constexpr int kDxTok = 32, kDxCols = 256;

template <typename T, int KT>  // KT = k when 1 or 2, 0 = generic k <= 8
__global__ void __launch_bounds__(256) dx_tiled_kernel(const T* __restrict__ dXe, const int* __restrict__ idx,
                                                       const int* __restrict__ slot,
                                                       const float* __restrict__ dL,
                                                       const float* __restrict__ Wg, int Tn, int k, int d,
                                                       int E, int C, int n, int Cm, T* __restrict__ dX) {
  extern __shared__ float dsm[];
  float* sW = dsm;                     // [E][kDxCols]
  float* sL = dsm + E * kDxCols;       // [kDxTok][E]
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * kDxCols;
  const int t0 = blockIdx.y * kDxTok;
  // the gathers do not depend on shared memory: issue them before staging
  const int cg = tid & 31, tg = tid >> 5;  // 32 column groups x 8 token groups
  const int col = c0 + cg * 8;
  float acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[i][c] = 0.f;
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
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      if (sl[i][j] < 0) continue;
      const T* src = dXe + send_row(ex[i][j], sl[i][j], E, C, n, Cm) * d + col;
      float x[8];
      if constexpr (sizeof(T) == 2) {
        load16(src, x, (const __nv_bfloat16*)nullptr);
      } else {
        load16(src, x, (const float*)nullptr);
        load16(src + 4, x + 4, (const float*)nullptr);
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[i][c] += x[c];
    }
  }
  for (int i = tid; i < E * kDxCols; i += 256) {
    const int col = i / E, e = i % E;  // coalesced read of Wg rows
    sW[e * kDxCols + col] = (c0 + col < d) ? Wg[(size_t)(c0 + col) * E + e] : 0.f;
  }
  for (int i = tid; i < kDxTok * E; i += 256) {
    const int r = i / E, e = i % E;
    sL[i] = (t0 + r < Tn) ? dL[(size_t)(t0 + r) * E + e] : 0.f;
  }
  __syncthreads();
  if (col >= d) return;
  // + dL · Wgᵀ
  for (int e = 0; e < E; ++e) {
    const float4 w0 = *reinterpret_cast<const float4*>(sW + e * kDxCols + cg * 8);
    const float4 w1 = *reinterpret_cast<const float4*>(sW + e * kDxCols + cg * 8 + 4);
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

// part[split][col][e] over tokens t = split*tps + lane + 8*i (8 token lanes = 8 warps,
// combined in shared memory in a fixed order).
template <typename T>
__global__ void __launch_bounds__(256) dwg_tiled_kernel(const T* __restrict__ X, const float* __restrict__ dL,
                                                        int Tn, int d, int E, int tps,
                                                        float* __restrict__ part) {
  __shared__ float red[4][256 * 8];
  const int tid = threadIdx.x;
  const int cg = tid & 31, lane_t = tid >> 5;
  const int col = blockIdx.x * 256 + cg * 8;
  const int split = blockIdx.y;
  const int e0 = blockIdx.z * 8;
  const int ne = min(8, E - e0);
  const int ta = split * tps, tb = min(Tn, ta + tps);
  float acc[8][8];
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[c][q] = 0.f;
  if (col < d) {
#pragma unroll 4
    for (int t = ta + lane_t; t < tb; t += 8) {
      float x[8];
      const T* src = X + (size_t)t * d + col;
      if constexpr (sizeof(T) == 2) {
        load16(src, x, (const __nv_bfloat16*)nullptr);
      } else {
        load16(src, x, (const float*)nullptr);
        load16(src + 4, x + 4, (const float*)nullptr);
      }
      float l[8];
      const float* lp = dL + (size_t)t * E + e0;
      if (ne == 8 && (E & 3) == 0) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(lp));
        const float4 b = __ldg(reinterpret_cast<const float4*>(lp + 4));
        l[0] = a.x; l[1] = a.y; l[2] = a.z; l[3] = a.w; l[4] = b.x; l[5] = b.y; l[6] = b.z; l[7] = b.w;
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) l[q] = q < ne ? __ldg(lp + q) : 0.f;
      }
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[c][q] = fmaf(x[c], l[q], acc[c][q]);
    }
  }
  // fixed-order tree over the 8 token lanes: (0+4,1+5,2+6,3+7), (0+2,1+3), (0+1)
  for (int half = 4; half >= 1; half >>= 1) {
    if (lane_t >= half && lane_t < 2 * half) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int q = 0; q < 8; ++q) red[lane_t - half][(c * 8 + q) * 32 + cg] = acc[c][q];
    }
    __syncthreads();
    if (lane_t < half) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[c][q] += red[lane_t][(c * 8 + q) * 32 + cg];
    }
    __syncthreads();
  }
  if (lane_t == 0 && col < d) {
    float* dst = part + ((size_t)split * d + col) * E + e0;
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < ne) dst[(size_t)c * E + q] = acc[c][q];
  }
}

__global__ void dwg_reduce_kernel(const float* __restrict__ part, int nparts, int dE,
                                  float* __restrict__ dWg) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= dE) return;
  float s = 0.f;
  int q = 0;
  for (; q + 8 <= nparts; q += 8) {  // 8 independent loads in flight, summed in order
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(part + (size_t)(q + u) * dE + i);
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; q < nparts; ++q) s += part[(size_t)q * dE + i];
  dWg[i] = s;
}

int dwg_splits(int T, int d, int E) {
  const int dblk = (d + 255) / 256, eblk = (E + 7) / 8;
  int want = (1200 + dblk * eblk - 1) / (dblk * eblk);  // ~8 waves of CTAs
  const int maxs = (T + 127) / 128;                      // >= 16 tokens per token lane
  if (want > maxs) want = maxs;
  return want < 1 ? 1 : want;
}

}  // namespace

size_t dwg_scratch_floats(int T, int d, int E) {
  return (size_t)dwg_splits(T, d, E) * d * E;
}

template <typename T, int KT>
static void launch_dx_t(const void* dXe, const int* idx, const int* slot, const float* dL,
                        const float* Wg, int Tn, int k, int d, int E, int C, int n, int Cm, void* dX,
                        cudaStream_t s) {
  dim3 grid((d + kDxCols - 1) / kDxCols, (Tn + kDxTok - 1) / kDxTok);
  const size_t smem = sizeof(float) * ((size_t)E * kDxCols + kDxTok * E);
  static bool set = false;
  if (!set) {
    LINA_CUDA_CHECK(cudaFuncSetAttribute(dx_tiled_kernel<T, KT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    set = true;
  }
  dx_tiled_kernel<T, KT><<<grid, 256, smem, s>>>((const T*)dXe, idx, slot, dL, Wg, Tn, k, d, E, C, n, Cm,
                                                (T*)dX);
}

void launch_dx(int dtype, const void* dXe, const int* idx, const int* slot, const float* dL,
               const float* Wg, int T, int k, int d, int E, int C, int n, int Cm, void* dX,
               cudaStream_t s) {
  if (T <= 0) return;
  auto go = [&](auto tag) {
    using ET = decltype(tag);
    if (k == 1) launch_dx_t<ET, 1>(dXe, idx, slot, dL, Wg, T, k, d, E, C, n, Cm, dX, s);
    else if (k == 2) launch_dx_t<ET, 2>(dXe, idx, slot, dL, Wg, T, k, d, E, C, n, Cm, dX, s);
    else launch_dx_t<ET, 0>(dXe, idx, slot, dL, Wg, T, k, d, E, C, n, Cm, dX, s);
  };
  if (dtype == 0) go(float{});
  else go(__nv_bfloat16{});
  LINA_LAUNCH_CHECK();
}

void launch_dwg(int dtype, const void* X, const float* dL, int T, int d, int E, float* scratch,
                float* dWg, cudaStream_t s) {
  if (T <= 0) {
    LINA_CUDA_CHECK(cudaMemsetAsync(dWg, 0, sizeof(float) * (size_t)d * E, s));
    return;
  }
  const int nsplit = dwg_splits(T, d, E);
  const int tps = (T + nsplit - 1) / nsplit;
  dim3 grid((d + 255) / 256, nsplit, (E + 7) / 8);
  if (dtype == 0)
    dwg_tiled_kernel<float><<<grid, 256, 0, s>>>((const float*)X, dL, T, d, E, tps, scratch);
  else
    dwg_tiled_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)X, dL, T, d, E, tps,
                                                         scratch);
  LINA_LAUNCH_CHECK();
  const int dE = d * E;
  dwg_reduce_kernel<<<(dE + 255) / 256, 256, 0, s>>>(scratch, nsplit, dE, dWg);
  LINA_LAUNCH_CHECK();
}

}  // namespace lina
