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
// threads owns BT=32 tokens x all E experts; the d reduction runs in 64/128-column
// slabs staged in shared memory (X transposed to fp32, Wg slab), each thread
// keeping one token x E/8 experts in registers.  Each logit is one fp32 FMA chain in ascending d
// order: deterministic, and exact for the grid inputs of DESIGN.md §4.  The
// epilogue keeps logits in shared memory and gives one warp per token for the
// softmax (warp-shuffle max/sum) and k rounds of warp arg-max.
#include <math.h>

#include "../common.h"
#include "../kernels.h"

namespace lina {
namespace {

constexpr int kGateBT = 32;

__device__ __forceinline__ bool key_better(float la, int ia, float lb, int ib) {
  return la > lb || (la == lb && ia < ib);
}

// EP = padded expert count (8/16/32/64).  Threads: 8 along experts (TE = EP/8 each) x
// 32 along tokens (one token each).  DK-column slabs of X (transposed to fp32) and Wg
// are double-buffered through registers: the global loads of slab i+1 are issued
// before the FMAs of slab i, so each CTA keeps its next 4 KB-8 KB in flight.
template <typename TIn, int EP>
__global__ void __launch_bounds__(256) gate_topk_kernel(const TIn* __restrict__ X,
                                                        const float* __restrict__ Wg, int T, int d,
                                                        int E, int k, int write_routing,
                                                        float* __restrict__ probs,
                                                        int* __restrict__ idx,
                                                        float* __restrict__ gate) {
  constexpr int BT = kGateBT;
  constexpr int DK = (EP <= 16) ? 128 : 64;
  constexpr int TE = EP / 8;
  constexpr int XV = BT * DK / 256;        // X elements per thread per slab (16 or 8)
  constexpr int WV = DK * EP / 256;        // Wg floats per thread per slab
  __shared__ float xs[DK][BT + 1];
  __shared__ float ws[DK][EP];
  __shared__ float lt[BT][EP + 1];

  const int tid = threadIdx.x;
  const int tx = tid & 7, ty = tid >> 3;   // expert group, token
  const int t0 = blockIdx.x * BT;
  // slab loaders: X row r = tid / (DK/XV), columns cs..cs+XV; Wg flat index tid*WV..
  constexpr int XT = DK / XV;              // threads per X row
  const int xr = tid / XT, xc = (tid % XT) * XV;
  float xreg[XV], wreg[WV];
  auto load_slab = [&](int k0) {
    const int t = t0 + xr;
#pragma unroll
    for (int i = 0; i < XV; i += 8) {
      const int c = k0 + xc + i;
      if (t < T && c + 8 <= d && ((d * (int)sizeof(TIn)) % 16 == 0)) {
        const TIn* src = X + (size_t)t * d + c;
        if constexpr (sizeof(TIn) == 2) {
          load16(src, xreg + i, (const __nv_bfloat16*)nullptr);
        } else {
          load16(src, xreg + i, (const float*)nullptr);
          load16(src + 4, xreg + i + 4, (const float*)nullptr);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          xreg[i + q] = (t < T && c + q < d) ? Elt<TIn>::to_f(X[(size_t)t * d + c + q]) : 0.f;
      }
    }
#pragma unroll
    for (int i = 0; i < WV; ++i) {
      const int f = tid * WV + i;
      const int kk = f / EP, e = f % EP;
      wreg[i] = (e < E && k0 + kk < d) ? __ldg(Wg + (size_t)(k0 + kk) * E + e) : 0.f;
    }
  };
  auto store_slab = [&]() {
#pragma unroll
    for (int i = 0; i < XV; ++i) xs[xc + i][xr] = xreg[i];
#pragma unroll
    for (int i = 0; i < WV; ++i) {
      const int f = tid * WV + i;
      ws[f / EP][f % EP] = wreg[i];
    }
  };
  float acc[TE];
#pragma unroll
  for (int e = 0; e < TE; ++e) acc[e] = 0.f;
  load_slab(0);
  for (int k0 = 0; k0 < d; k0 += DK) {
    store_slab();
    __syncthreads();
    if (k0 + DK < d) load_slab(k0 + DK);   // in flight during the FMAs below
#pragma unroll 8
    for (int kk = 0; kk < DK; ++kk) {
      const float a = xs[kk][ty];
#pragma unroll
      for (int e = 0; e < TE; ++e) acc[e] = fmaf(a, ws[kk][tx * TE + e], acc[e]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int e = 0; e < TE; ++e) lt[ty][tx * TE + e] = acc[e];
  __syncthreads();

  const int warp = tid >> 5, lane = tid & 31;
  for (int r = warp; r < kGateBT; r += 8) {
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
