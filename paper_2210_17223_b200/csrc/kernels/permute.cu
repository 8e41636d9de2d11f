// S3 permute (K3), S7 combine (K7) and their backward (S8 a, e, f) — the HBM-bound
// row movers around the expert GEMMs.
//
// Buffer layout shared by all of them ("chunk-major send layout"):
//   Send[n][E][Cm][w] with Cm = ceil(C/n); chunk c holds capacity slots
//   [b_c, b_{c+1}) of every expert (R10), rows beyond the chunk or beyond the
//   kept count are zero.  For a static placement (experts of rank r are
//   [r*E_l, (r+1)*E_l)), chunk c's block for peer r is contiguous, so one
//   equal-split all-to-all per chunk moves it.
//
// permute       : Send[row] = X[t] for the assignment holding that slot, else 0
//                 ("dispatches the token" P:98, first all-to-all P:132).
// combine       : y_t = sum_{j kept, ascending} g_tj * Recv[row(t,j)]  (fp32 acc, R9)
//                 ("reshaping the tensors and computing the weighted output" P:172-173).
// combine_bwd   : dg_tj = <dY_t, O_tj>,  dSend[row] = g_tj * dY_t  (else 0).
// gate_bwd      : dL_t = p ∘ (dp − <p,dp>),  dp from dg through g (R13).
// dx            : dX_t = sum_{j kept} dXe[row(t,j)] + sum_e dL_te Wg[:,e].
// dwg           : dWg = Xᵀ dL, split over token ranges, reduced in fixed order.
// Rows are moved as 16-byte vectors, one warp per row / token.
#include "../common.h"
#include "../kernels.h"

namespace lina {
namespace {

__device__ __forceinline__ size_t send_row(int e, int s, int E, int C, int n, int Cm) {
  const int c = chunk_of(s, C, n);
  return ((size_t)c * E + e) * Cm + (s - chunk_begin(c, C, n));
}

template <typename T>
__global__ void permute_kernel(const T* __restrict__ X, const int* __restrict__ tok_of, int k,
                               int d, int E, int C, int n, int Cm, T* __restrict__ Send) {
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long rows = (long long)n * E * Cm;
  if (gw >= rows) return;
  const int r = (int)(gw % Cm);
  const int ce = (int)(gw / Cm);
  const int e = ce % E, c = ce / E;
  const int b = chunk_begin(c, C, n), Cc = chunk_begin(c + 1, C, n) - b;
  const int a = (r < Cc) ? tok_of[(size_t)e * C + b + r] : -1;
  constexpr int V = 16 / sizeof(T);
  uint4* dst = reinterpret_cast<uint4*>(Send + (size_t)gw * d);
  const int nv = d / V;
  if (a >= 0) {
    const uint4* src = reinterpret_cast<const uint4*>(X + (size_t)(a / k) * d);
    for (int v = lane; v < nv; v += 32) dst[v] = src[v];
  } else {
    for (int v = lane; v < nv; v += 32) dst[v] = make_uint4(0, 0, 0, 0);
  }
}

template <typename T>
__global__ void combine_kernel(const T* __restrict__ Recv, const int* __restrict__ idx,
                               const int* __restrict__ slot, const float* __restrict__ gate,
                               int Tn, int k, int d, int E, int C, int n, int Cm,
                               T* __restrict__ Y) {
  const long long t = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= Tn) return;
  constexpr int V = 16 / sizeof(T);
  const T* rowp[8];
  float g[8];
  int kk = 0;
  for (int j = 0; j < k; ++j) {
    const int s = slot[t * k + j];
    if (s >= 0) {
      rowp[kk] = Recv + send_row(idx[t * k + j], s, E, C, n, Cm) * d;
      g[kk] = gate[t * k + j];
      ++kk;
    }
  }
  for (int v = lane; v < d / V; v += 32) {
    float acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0.f;
    for (int q = 0; q < kk; ++q) {
      float x[V];
      load16(rowp[q] + v * V, x, (const T*)nullptr);
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] = fmaf(g[q], x[i], acc[i]);
    }
    store16(Y + t * d + v * V, acc, (T*)nullptr);
  }
}

template <typename T>
__global__ void combine_bwd_kernel(const T* __restrict__ dY, const T* __restrict__ Recv,
                                   const int* __restrict__ tok_of, const float* __restrict__ gate,
                                   int k, int d, int E, int C, int n, int Cm,
                                   T* __restrict__ dSend, float* __restrict__ dg) {
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long rows = (long long)n * E * Cm;
  if (gw >= rows) return;
  const int r = (int)(gw % Cm);
  const int ce = (int)(gw / Cm);
  const int e = ce % E, c = ce / E;
  const int b = chunk_begin(c, C, n), Cc = chunk_begin(c + 1, C, n) - b;
  const int a = (r < Cc) ? tok_of[(size_t)e * C + b + r] : -1;
  constexpr int V = 16 / sizeof(T);
  const int nv = d / V;
  T* dst = dSend + (size_t)gw * d;
  if (a < 0) {
    for (int v = lane; v < nv; v += 32) reinterpret_cast<uint4*>(dst)[v] = make_uint4(0, 0, 0, 0);
    return;
  }
  const float g = gate[a];
  const T* dy = dY + (size_t)(a / k) * d;
  const T* o = Recv + (size_t)gw * d;
  float dot = 0.f;
  for (int v = lane; v < nv; v += 32) {
    float x[V], w[V];
    load16(dy + v * V, x, (const T*)nullptr);
    load16(o + v * V, w, (const T*)nullptr);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      dot = fmaf(x[i], w[i], dot);
      x[i] *= g;
    }
    store16(dst + v * V, x, (T*)nullptr);
  }
#pragma unroll
  for (int o2 = 16; o2; o2 >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o2);
  if (lane == 0) dg[a] = dot;
}

// dL for one token per warp.  k=1: g0 = p_e0  => dp_e0 = dg0.
// k>=2: g_j = p_ej / S  =>  dp_ei = (dg_i − Σ_j g_j dg_j) / S.   dL = p ∘ (dp − <p,dp>).
__global__ void gate_bwd_kernel(const float* __restrict__ probs, const int* __restrict__ idx,
                                const float* __restrict__ gate, const float* __restrict__ dg,
                                int Tn, int k, int E, float* __restrict__ dL) {
  const long long t = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= Tn) return;
  const float p0 = lane < E ? probs[t * E + lane] : 0.f;
  const float p1 = lane + 32 < E ? probs[t * E + lane + 32] : 0.f;
  float dp0 = 0.f, dp1 = 0.f;
  if (k == 1) {
    const int e0 = idx[t];
    if (e0 == lane) dp0 = dg[t];
    if (e0 == lane + 32) dp1 = dg[t];
  } else {
    float S = 0.f, sgd = 0.f;
    for (int j = 0; j < k; ++j) {
      const int e = idx[t * k + j];
      S += probs[t * E + e];
      sgd = fmaf(gate[t * k + j], dg[t * k + j], sgd);
    }
    for (int j = 0; j < k; ++j) {
      const int e = idx[t * k + j];
      const float v = (dg[t * k + j] - sgd) / S;
      if (e == lane) dp0 = v;
      if (e == lane + 32) dp1 = v;
    }
  }
  float dot = p0 * dp0 + p1 * dp1;
#pragma unroll
  for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  if (lane < E) dL[t * E + lane] = p0 * (dp0 - dot);
  if (lane + 32 < E) dL[t * E + lane + 32] = p1 * (dp1 - dot);
}

// dX = gather-sum of returned expert input-gradients + dL · Wgᵀ.
// CTA: 64 tokens x 64 columns per step; dL tile and a transposed Wg slab in smem.
template <typename T>
__global__ void __launch_bounds__(256) dx_kernel(const T* __restrict__ dXe, const int* __restrict__ idx,
                                                 const int* __restrict__ slot,
                                                 const float* __restrict__ dL,
                                                 const float* __restrict__ Wg, int Tn, int k, int d,
                                                 int E, int C, int n, int Cm, T* __restrict__ dX) {
  __shared__ float sL[64][65];
  __shared__ float sW[64][68];  // [e][col]
  const int tid = threadIdx.x;
  const int t0 = blockIdx.x * 64;
  for (int i = tid; i < 64 * E; i += 256) {
    const int r = i / E, e = i % E;
    sL[r][e] = (t0 + r < Tn) ? dL[(size_t)(t0 + r) * E + e] : 0.f;
  }
  const int r = tid >> 2;          // token row in tile
  const int cq = (tid & 3) * 16;   // 16 columns per thread
  const int t = t0 + r;
  size_t rows[8];
  int kk = 0;
  if (t < Tn)
    for (int j = 0; j < k; ++j) {
      const int s = slot[(size_t)t * k + j];
      if (s >= 0) rows[kk++] = send_row(idx[(size_t)t * k + j], s, E, C, n, Cm);
    }
  for (int c0 = 0; c0 < d; c0 += 64) {
    __syncthreads();
    for (int i = tid; i < 64 * E; i += 256) {
      const int col = i / E, e = i % E;
      sW[e][col] = (c0 + col < d) ? Wg[(size_t)(c0 + col) * E + e] : 0.f;
    }
    __syncthreads();
    if (t >= Tn || c0 + cq >= d) continue;
    float acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.f;
    for (int q = 0; q < kk; ++q) {
      const T* src = dXe + rows[q] * d + c0 + cq;
      constexpr int V = 16 / sizeof(T);
#pragma unroll
      for (int v = 0; v < 16 / V; ++v) {
        float x[V];
        load16(src + v * V, x, (const T*)nullptr);
#pragma unroll
        for (int i = 0; i < V; ++i) acc[v * V + i] += x[i];
      }
    }
    for (int e = 0; e < E; ++e) {
      const float l = sL[r][e];
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fmaf(l, sW[e][cq + i], acc[i]);
    }
    constexpr int V = 16 / sizeof(T);
#pragma unroll
    for (int v = 0; v < 16 / V; ++v) store16(dX + (size_t)t * d + c0 + cq + v * V, acc + v * V, (T*)nullptr);
  }
}

// Partial dWg over a token range: part[split][i][e] = Σ_{t in split} X[t][i] dL[t][e].
template <typename T>
__global__ void __launch_bounds__(256) dwg_partial_kernel(const T* __restrict__ X,
                                                          const float* __restrict__ dL, int Tn,
                                                          int d, int E, int tok_per_split,
                                                          float* __restrict__ part) {
  __shared__ float sX[32][65];  // [tok][col]
  __shared__ float sL[32][65];  // [tok][e]
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * 64;
  const int split = blockIdx.y;
  const int ta = split * tok_per_split;
  const int tb = min(Tn, ta + tok_per_split);
  // thread owns column (tid & 63) and experts e = (tid >> 6) + 4*q
  const int col = tid & 63, eg = tid >> 6;
  float acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.f;
  for (int tt = ta; tt < tb; tt += 32) {
    __syncthreads();
    for (int i = tid; i < 32 * 64; i += 256) {
      const int r = i / 64, c = i % 64;
      sX[r][c] = (tt + r < tb && c0 + c < d) ? Elt<T>::to_f(X[(size_t)(tt + r) * d + c0 + c]) : 0.f;
    }
    for (int i = tid; i < 32 * E; i += 256) {
      const int r = i / E, e = i % E;
      sL[r][e] = (tt + r < tb) ? dL[(size_t)(tt + r) * E + e] : 0.f;
    }
    __syncthreads();
    for (int r = 0; r < 32; ++r) {
      const float x = sX[r][col];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int e = eg + 4 * q;
        if (e < E) acc[q] = fmaf(x, sL[r][e], acc[q]);
      }
    }
  }
  if (c0 + col < d)
    for (int q = 0; q < 16; ++q) {
      const int e = eg + 4 * q;
      if (e < E) part[((size_t)split * d + c0 + col) * E + e] = acc[q];
    }
}

__global__ void dwg_reduce_kernel(const float* __restrict__ part, int nsplit, int dE,
                                  float* __restrict__ dWg) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= dE) return;
  float s = 0.f;
  for (int q = 0; q < nsplit; ++q) s += part[(size_t)q * dE + i];
  dWg[i] = s;
}

inline int blocks_for_warps(long long warps, int threads = 256) {
  return (int)((warps * 32 + threads - 1) / threads);
}

}  // namespace

constexpr int kDwgTokPerSplit = 512;

size_t dwg_scratch_floats(int T, int d, int E) {
  const int nsplit = (T + kDwgTokPerSplit - 1) / kDwgTokPerSplit;
  return (size_t)(nsplit > 0 ? nsplit : 1) * d * E;
}

#define LINA_DISPATCH_T(dtype, ...)                 \
  do {                                              \
    if ((dtype) == 0) {                             \
      using ET = float;                              \
      __VA_ARGS__;                                  \
    } else {                                        \
      using ET = __nv_bfloat16;                      \
      __VA_ARGS__;                                  \
    }                                               \
  } while (0)

void launch_permute(int dtype, const void* X, const int* tok_of, int k, int d, int E, int C, int n,
                    int Cm, void* Send, cudaStream_t s) {
  const long long rows = (long long)n * E * Cm;
  if (rows == 0) return;
  LINA_DISPATCH_T(dtype, permute_kernel<ET><<<blocks_for_warps(rows), 256, 0, s>>>(
                             (const ET*)X, tok_of, k, d, E, C, n, Cm, (ET*)Send));
  LINA_LAUNCH_CHECK();
}

void launch_combine(int dtype, const void* Recv, const int* idx, const int* slot, const float* gate,
                    int T, int k, int d, int E, int C, int n, int Cm, void* Y, cudaStream_t s) {
  if (T <= 0) return;
  LINA_DISPATCH_T(dtype, combine_kernel<ET><<<blocks_for_warps(T), 256, 0, s>>>(
                             (const ET*)Recv, idx, slot, gate, T, k, d, E, C, n, Cm, (ET*)Y));
  LINA_LAUNCH_CHECK();
}

void launch_combine_bwd(int dtype, const void* dY, const void* Recv, const int* tok_of,
                        const float* gate, int T, int k, int d, int E, int C, int n, int Cm,
                        void* dSend, float* dg, cudaStream_t s) {
  if (T > 0) LINA_CUDA_CHECK(cudaMemsetAsync(dg, 0, sizeof(float) * (size_t)T * k, s));
  const long long rows = (long long)n * E * Cm;
  if (rows == 0) return;
  LINA_DISPATCH_T(dtype, combine_bwd_kernel<ET><<<blocks_for_warps(rows), 256, 0, s>>>(
                             (const ET*)dY, (const ET*)Recv, tok_of, gate, k, d, E, C, n, Cm,
                             (ET*)dSend, dg));
  LINA_LAUNCH_CHECK();
}

void launch_gate_bwd(const float* probs, const int* idx, const float* gate, const float* dg, int T,
                     int k, int E, float* dL, cudaStream_t s) {
  if (T <= 0) return;
  gate_bwd_kernel<<<blocks_for_warps(T), 256, 0, s>>>(probs, idx, gate, dg, T, k, E, dL);
  LINA_LAUNCH_CHECK();
}

void launch_dx(int dtype, const void* dXe, const int* idx, const int* slot, const float* dL,
               const float* Wg, int T, int k, int d, int E, int C, int n, int Cm, void* dX,
               cudaStream_t s) {
  if (T <= 0) return;
  LINA_DISPATCH_T(dtype, dx_kernel<ET><<<(T + 63) / 64, 256, 0, s>>>(
                             (const ET*)dXe, idx, slot, dL, Wg, T, k, d, E, C, n, Cm, (ET*)dX));
  LINA_LAUNCH_CHECK();
}

void launch_dwg(int dtype, const void* X, const float* dL, int T, int d, int E, float* scratch,
                float* dWg, cudaStream_t s) {
  if (T <= 0) {
    LINA_CUDA_CHECK(cudaMemsetAsync(dWg, 0, sizeof(float) * (size_t)d * E, s));
    return;
  }
  const int nsplit = (T + kDwgTokPerSplit - 1) / kDwgTokPerSplit;
  dim3 grid((d + 63) / 64, nsplit);
  LINA_DISPATCH_T(dtype, dwg_partial_kernel<ET><<<grid, 256, 0, s>>>((const ET*)X, dL, T, d, E,
                                                                     kDwgTokPerSplit, scratch));
  LINA_LAUNCH_CHECK();
  const int dE = d * E;
  dwg_reduce_kernel<<<(dE + 255) / 256, 256, 0, s>>>(scratch, nsplit, dE, dWg);
  LINA_LAUNCH_CHECK();
}

}  // namespace lina
