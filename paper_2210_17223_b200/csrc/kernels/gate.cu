// S1 (K1): fused gate GEMM + softmax + top-k + gate weights.
//
// PAPER.md:98 (§2.1): "The gating network takes in the embedding vector of each
// token and multiplies them with its trainable matrix. Based on the results, it
// dispatches the token to a small number of experts (usually one or two)."
// Readings: no bias/noise and softmax over all E (R1); fp32 logits/probabilities
// (R2); top-k keyed on the logits, ties to the lower expert id (R3); k=1 gate is
// the raw probability, k>=2 renormalised over the k selected (R4).
//
// Layout: X [T,d] (bf16|fp32) row-major, Wg [d,E] fp32 row-major.  One CTA of 256
// threads owns BT=64 tokens x all E experts; the d reduction runs in DK=32 slabs
// staged in shared memory (X transposed to fp32, Wg slab), each thread keeping a
// TM x TE register micro-tile.  Each logit is one fp32 FMA chain in ascending d
// order: deterministic, and exact for the grid inputs of DESIGN.md §4.  The
// epilogue keeps logits in shared memory and gives one warp per token for the
// softmax (warp-shuffle max/sum) and k rounds of warp arg-max.
#include <math.h>

#include "../common.h"
#include "../kernels.h"

namespace lina {
namespace {

constexpr int kGateBT = 64;
constexpr int kGateDK = 32;

__device__ __forceinline__ bool key_better(float la, int ia, float lb, int ib) {
  return la > lb || (la == lb && ia < ib);
}

template <typename TIn, int EP>
__global__ void __launch_bounds__(256) gate_topk_kernel(const TIn* __restrict__ X,
                                                        const float* __restrict__ Wg, int T, int d,
                                                        int E, int k, int write_routing,
                                                        float* __restrict__ probs,
                                                        int* __restrict__ idx,
                                                        float* __restrict__ gate) {
  constexpr int BT = kGateBT, DK = kGateDK;
  constexpr int TE = (EP >= 16) ? 4 : 2;
  constexpr int TX = EP / TE;
  constexpr int TY = 256 / TX;
  constexpr int TM = BT / TY;
  static_assert(TM >= 1 && TM * TY == BT, "tile");
  __shared__ float xs[DK][BT + 4];
  __shared__ float ws[DK][EP];
  __shared__ float lt[BT][EP + 1];

  const int tid = threadIdx.x;
  const int tx = tid % TX, ty = tid / TX;
  const int t0 = blockIdx.x * BT;
  float acc[TM][TE];
#pragma unroll
  for (int m = 0; m < TM; ++m)
#pragma unroll
    for (int e = 0; e < TE; ++e) acc[m][e] = 0.f;

  for (int k0 = 0; k0 < d; k0 += DK) {
    {  // X slab: 64 rows x 32 cols, 8 consecutive elements per thread
      const int r = tid >> 2, cs = (tid & 3) * 8;
      const int t = t0 + r;
      float v[8];
      if (t < T && k0 + cs + 8 <= d && ((d * sizeof(TIn)) % 16 == 0)) {
        const TIn* src = X + (size_t)t * d + k0 + cs;
        if constexpr (sizeof(TIn) == 2) {
          load16(src, v, (const __nv_bfloat16*)nullptr);
        } else {
          load16(src, v, (const float*)nullptr);
          load16(src + 4, v + 4, (const float*)nullptr);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          v[i] = (t < T && k0 + cs + i < d) ? Elt<TIn>::to_f(X[(size_t)t * d + k0 + cs + i]) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) xs[cs + i][r] = v[i];
    }
    for (int i = tid; i < DK * EP; i += 256) {
      const int kk = i / EP, e = i % EP;
      ws[kk][e] = (e < E && k0 + kk < d) ? Wg[(size_t)(k0 + kk) * E + e] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < DK; ++kk) {
      float a[TM], b[TE];
#pragma unroll
      for (int m = 0; m < TM; ++m) a[m] = xs[kk][ty * TM + m];
#pragma unroll
      for (int e = 0; e < TE; ++e) b[e] = ws[kk][tx * TE + e];
#pragma unroll
      for (int m = 0; m < TM; ++m)
#pragma unroll
        for (int e = 0; e < TE; ++e) acc[m][e] = fmaf(a[m], b[e], acc[m][e]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int m = 0; m < TM; ++m)
#pragma unroll
    for (int e = 0; e < TE; ++e) lt[ty * TM + m][tx * TE + e] = acc[m][e];
  __syncthreads();

  const int warp = tid >> 5, lane = tid & 31;
  for (int r = warp; r < BT; r += 8) {
    const int t = t0 + r;
    if (t >= T) break;
    const bool v0 = lane < E, v1 = lane + 32 < E;
    const float l0 = v0 ? lt[r][lane] : -INFINITY;
    const float l1 = v1 ? lt[r][lane + 32] : -INFINITY;
    float mx = fmaxf(l0, l1);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float z0 = v0 ? expf(l0 - mx) : 0.f;
    const float z1 = v1 ? expf(l1 - mx) : 0.f;
    float s = z0 + z1;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float p0 = z0 / s, p1 = z1 / s;
    if (v0) probs[(size_t)t * E + lane] = p0;
    if (v1) probs[(size_t)t * E + lane + 32] = p1;
    if (!write_routing) continue;
    // k rounds of warp arg-max on (logit desc, id asc)
    bool sel0 = !v0, sel1 = !v1;
    float psel[8];
    float psum = 0.f;
    for (int j = 0; j < k; ++j) {
      float bl = -INFINITY;
      int bi = 0x7fffffff;
      if (!sel0) { bl = l0; bi = lane; }
      if (!sel1 && key_better(l1, lane + 32, bl, bi)) { bl = l1; bi = lane + 32; }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const float ol = __shfl_xor_sync(0xffffffffu, bl, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (key_better(ol, oi, bl, bi)) { bl = ol; bi = oi; }
      }
      // owner lane marks it; broadcast its probability
      float pw = 0.f;
      if (bi == lane) { sel0 = true; pw = p0; }
      if (bi == lane + 32) { sel1 = true; pw = p1; }
      const int owner = bi & 31;
      pw = __shfl_sync(0xffffffffu, pw, owner);
      psel[j] = pw;
      psum += pw;
      if (lane == 0) idx[(size_t)t * k + j] = bi;
    }
    if (lane == 0) {
      for (int j = 0; j < k; ++j) gate[(size_t)t * k + j] = (k == 1) ? psel[0] : psel[j] / psum;
    }
  }
}

template <typename TIn, int EP>
void launch_gate_ep(const void* X, const float* Wg, int T, int d, int E, int k, int write_routing,
                    float* probs, int* idx, float* gate, cudaStream_t s) {
  const int blocks = (T + kGateBT - 1) / kGateBT;
  gate_topk_kernel<TIn, EP><<<blocks, 256, 0, s>>>((const TIn*)X, Wg, T, d, E, k, write_routing,
                                                    probs, idx, gate);
}

}  // namespace

void launch_gate_topk(int dtype, const void* X, const float* Wg, int T, int d, int E, int k,
                      int write_routing, float* probs, int* idx, float* gate, cudaStream_t s) {
  if (T <= 0) return;
  auto go = [&](auto tag) {
    using TIn = decltype(tag);
    if (E <= 8) launch_gate_ep<TIn, 8>(X, Wg, T, d, E, k, write_routing, probs, idx, gate, s);
    else if (E <= 16) launch_gate_ep<TIn, 16>(X, Wg, T, d, E, k, write_routing, probs, idx, gate, s);
    else if (E <= 32) launch_gate_ep<TIn, 32>(X, Wg, T, d, E, k, write_routing, probs, idx, gate, s);
    else launch_gate_ep<TIn, 64>(X, Wg, T, d, E, k, write_routing, probs, idx, gate, s);
  };
  if (dtype == 0) go(float{});
  else go(__nv_bfloat16{});
  LINA_LAUNCH_CHECK();
}

}  // namespace lina
