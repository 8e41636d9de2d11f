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
// (dX and dWg are in gate_bwd.cu.)
// Rows are moved as 16-byte vectors, one warp per row / token.
#include "../common.h"
#include "../kernels.h"

namespace lina {
namespace {

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
  const int b = chunk_begin_p(c, C, Cm), Cc = chunk_begin_p(c + 1, C, Cm) - b;
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
#pragma unroll 4
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
  const int b = chunk_begin_p(c, C, Cm), Cc = chunk_begin_p(c + 1, C, Cm) - b;
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

// ---- fused dispatch: the same row loops, but each row is stored straight into the
// owner's receive buffer over NVLink (peer[o] = rank o's buffer mapped here).  Row
// (c, e, r) of the send layout lands at recv row ((c*P + me)*El + e%El)*Cm + r of
// owner o = e / El: the permute IS the dispatch all-to-all.
__device__ __forceinline__ size_t peer_row(int c, int e, int r, int El, int P, int me, int Cm) {
  return (((size_t)c * P + me) * El + (e % El)) * Cm + r;
}

template <typename T>
__global__ void permute_peer_kernel(const T* __restrict__ X, const int* __restrict__ tok_of, int k,
                                    int d, int E, int C, int n, int Cm, int El, int P, int me,
                                    T* const* __restrict__ peer) {
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long rows = (long long)n * E * Cm;
  if (gw >= rows) return;
  const int r = (int)(gw % Cm);
  const int ce = (int)(gw / Cm);
  const int e = ce % E, c = ce / E;
  const int b = chunk_begin_p(c, C, Cm), Cc = chunk_begin_p(c + 1, C, Cm) - b;
  const int a = (r < Cc) ? tok_of[(size_t)e * C + b + r] : -1;
  constexpr int V = 16 / sizeof(T);
  uint4* dst = reinterpret_cast<uint4*>(peer[e / El] + peer_row(c, e, r, El, P, me, Cm) * d);
  const int nv = d / V;
  if (a >= 0) {
    const uint4* src = reinterpret_cast<const uint4*>(X + (size_t)(a / k) * d);
    for (int v = lane; v < nv; v += 32) dst[v] = src[v];
  } else {
    for (int v = lane; v < nv; v += 32) dst[v] = make_uint4(0, 0, 0, 0);
  }
}

template <typename T>
__global__ void combine_bwd_peer_kernel(const T* __restrict__ dY, const T* __restrict__ Recv,
                                        const int* __restrict__ tok_of, const float* __restrict__ gate,
                                        int k, int d, int E, int C, int n, int Cm, int El, int P, int me,
                                        T* const* __restrict__ peer, float* __restrict__ dg) {
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long rows = (long long)n * E * Cm;
  if (gw >= rows) return;
  const int r = (int)(gw % Cm);
  const int ce = (int)(gw / Cm);
  const int e = ce % E, c = ce / E;
  const int b = chunk_begin_p(c, C, Cm), Cc = chunk_begin_p(c + 1, C, Cm) - b;
  const int a = (r < Cc) ? tok_of[(size_t)e * C + b + r] : -1;
  constexpr int V = 16 / sizeof(T);
  const int nv = d / V;
  T* dst = peer[e / El] + peer_row(c, e, r, El, P, me, Cm) * d;
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

// kept[o*El + el] (this source's counts for owner o's experts) -> owner's recv_kept[me*El + el]
__global__ void counts_peer_kernel(const int* __restrict__ kept, int El, int P, int me,
                                   int* const* __restrict__ peer) {
  for (int i = threadIdx.x; i < P * El; i += blockDim.x) {
    const int o = i / El, el = i % El;
    peer[o][me * El + el] = kept[i];
  }
}

inline int blocks_for_warps(long long warps, int threads = 256) {
  return (int)((warps * 32 + threads - 1) / threads);
}

}  // namespace

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

void launch_permute_peer(int dtype, const void* X, const int* tok_of, const int* kept, int k, int d,
                         int E, int C, int n, int Cm, int El, int P, int me, void* const* peer_rows,
                         void* const* peer_counts, cudaStream_t s) {
  counts_peer_kernel<<<1, 128, 0, s>>>(kept, El, P, me, (int* const*)peer_counts);
  LINA_LAUNCH_CHECK();
  const long long rows = (long long)n * E * Cm;
  if (rows == 0) return;
  LINA_DISPATCH_T(dtype, permute_peer_kernel<ET><<<blocks_for_warps(rows), 256, 0, s>>>(
                             (const ET*)X, tok_of, k, d, E, C, n, Cm, El, P, me, (ET* const*)peer_rows));
  LINA_LAUNCH_CHECK();
}

void launch_combine_bwd_peer(int dtype, const void* dY, const void* Recv, const int* tok_of,
                             const float* gate, int T, int k, int d, int E, int C, int n, int Cm, int El,
                             int P, int me, void* const* peer_rows, float* dg, cudaStream_t s) {
  if (T > 0) LINA_CUDA_CHECK(cudaMemsetAsync(dg, 0, sizeof(float) * (size_t)T * k, s));
  const long long rows = (long long)n * E * Cm;
  if (rows == 0) return;
  LINA_DISPATCH_T(dtype, combine_bwd_peer_kernel<ET><<<blocks_for_warps(rows), 256, 0, s>>>(
                             (const ET*)dY, (const ET*)Recv, tok_of, gate, k, d, E, C, n, Cm, El, P, me,
                             (ET* const*)peer_rows, dg));
  LINA_LAUNCH_CHECK();
}

}  // namespace lina
