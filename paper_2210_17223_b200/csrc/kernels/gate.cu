// S1 (K1): fused gate GEMM + softmax + top-k + gate weights.
//
// PAPER.md:98 (§2.1): "The gating network takes in the embedding vector of each
// token and multiplies them with its trainable matrix. Based on the results, it
// dispatches the token to a small number of experts (usually one or two)."
// Readings: no bias/noise and softmax over all E (R1); fp32 logits/probabilities
// (R2); top-k keyed on the logits, ties to the lower expert id (R3); k=1 gate is
// the raw probability, k>=2 renormalised over the k selected (R4).
//
// Layout: X [T,d] (bf16|fp32) row-major, Wg [d,E] fp32 row-major.
//
// bf16 tokens (gate_mma_kernel): the logits X·Wg are an N = E <= 64 GEMM.  Each warp
// owns 16 tokens and a quarter of d and runs mma.sync m16n8k16 (bf16 in, fp32
// accumulate) with the fp32 gate weight split exactly into three bf16 terms (w = hi +
// mid + lo, 24 = 3 x 8 significand bits), so the product is the fp32 logit up to
// accumulation order — exact for the grid inputs of DESIGN.md §4.  Tokens are read
// straight from global memory as 16-byte vectors (16 loads in flight per lane); K is
// permuted consistently in A and B so each 16-byte vector feeds two k-steps.  The
// split Wg is staged once per CTA in shared memory in B-fragment order.  (Not a
// tcgen05 GEMM: N = E is 8..64 and the kernel is bound by reading X once.)
// fp32 tokens (gate_simt_kernel, the C1 path): a register-tiled FMA version.
// Both end in the same epilogue: logits in shared memory, one warp per token for
// the softmax (warp-shuffle max/sum) and k rounds of warp arg-max.
#include <math.h>
#include <stdlib.h>

#include <algorithm>

#include "../common.h"
#include "../kernels.h"
#include "../signal.h"

namespace lina {
namespace {

__device__ __forceinline__ bool key_better(float la, int ia, float lb, int ib) {
  return la > lb || (la == lb && ia < ib);
}

// Softmax, top-k and gate weights for `nrows` tokens whose E logits are rows of `lt`
// (shared memory, pitch `ldl`), row r <-> token t0 + r.  Called by one full warp.
// The warp is cut into 32/W segments of W = pow2ceil(E) lanes (W = 32 and two
// logits per lane when E > 32), so 4 tokens are reduced at once when E <= 8:
// every shuffle stays inside its segment (xor offsets < W).
__device__ __forceinline__ void gate_epilogue_rows(const float* lt, int ldl, int nrows, int t0, int T,
                                                   int E, int k, int write_routing,
                                                   float* __restrict__ probs, int* __restrict__ idx,
                                                   float* __restrict__ gate) {
  const int lane = threadIdx.x & 31;
  int W = 1;
  while (W < E && W < 32) W <<= 1;
  const int TP = 32 / W;
  const int seg = lane / W, sl = lane % W;
  for (int r0 = 0; r0 < nrows; r0 += TP) {
    const int r = r0 + seg;
    const int t = t0 + r;
    const bool live = r < nrows && t < T;
    const float* lrow = lt + (size_t)(live ? r : 0) * ldl;
    const bool v0 = live && sl < E, v1 = live && sl + 32 < E;
    const float l0 = v0 ? lrow[sl] : -INFINITY;
    const float l1 = v1 ? lrow[sl + 32] : -INFINITY;
    float mx = fmaxf(l0, l1);
    for (int o = W >> 1; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float z0 = v0 ? expf(l0 - mx) : 0.f;
    const float z1 = v1 ? expf(l1 - mx) : 0.f;
    float sum = z0 + z1;
    for (int o = W >> 1; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float p0 = v0 ? z0 / sum : 0.f, p1 = v1 ? z1 / sum : 0.f;
    if (v0) probs[(size_t)t * E + sl] = p0;
    if (v1) probs[(size_t)t * E + sl + 32] = p1;
    if (!write_routing) continue;
    bool sel0 = !v0, sel1 = !v1;
    float psel[8];
    float psum = 0.f;
    for (int j = 0; j < k; ++j) {
      float bl = -INFINITY;
      int bi = 0x7fffffff;
      if (!sel0) { bl = l0; bi = sl; }
      if (!sel1 && key_better(l1, sl + 32, bl, bi)) { bl = l1; bi = sl + 32; }
      for (int o = W >> 1; o; o >>= 1) {
        const float ol = __shfl_xor_sync(0xffffffffu, bl, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (key_better(ol, oi, bl, bi)) { bl = ol; bi = oi; }
      }
      float pw = 0.f;
      if (bi == sl) { sel0 = true; pw = p0; }
      if (bi == sl + 32) { sel1 = true; pw = p1; }
      pw = __shfl_sync(0xffffffffu, pw, seg * W + ((bi & 0x7fffffff) % W));
      psel[j] = pw;
      psum += pw;
      if (live && sl == 0) idx[(size_t)t * k + j] = bi;
    }
    if (live && sl == 0)
      for (int j = 0; j < k; ++j) gate[(size_t)t * k + j] = (k == 1) ? psel[0] : psel[j] / psum;
  }
}

// ------------------------------------------------------------------ tensor-core gate (bf16 X)
// CTA = kGTT token tiles (16 tokens each) x kGKS K-split warps.  Wg is staged once per
// pass as ready-made B fragments: frag[split][n][kstep][lane] (uint2 = two packed bf16
// pairs), i.e. the exact hi/mid/lo decomposition computed once per CTA instead of in the
// inner loop, and read back with one conflict-free 8-byte LDS per fragment.  The K-split
// partial logits are summed in a fixed order (deterministic).
constexpr int kGTT = 2;                   // 16-token tiles per CTA
constexpr int kGKS = 4;                   // K-split warps per tile
constexpr int kGThreads = 32 * kGTT * kGKS;
constexpr int kGTok = 16 * kGTT;          // tokens per CTA
constexpr size_t kGStageBudget = 150 * 1024;

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void split3(float w, float& hi, float& mid, float& lo) {
  hi = __bfloat162float(__float2bfloat16_rn(w));
  const float r1 = w - hi;
  mid = __bfloat162float(__float2bfloat16_rn(r1));
  lo = r1 - mid;  // <= 8 significant bits: exact in bf16
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// NT = ceil(E/8) n-tiles of 8 experts; PB = 32-column blocks staged per pass (runtime).
template <int NT>
__global__ void __launch_bounds__(kGThreads) gate_mma_kernel(const __nv_bfloat16* __restrict__ X,
                                                             const float* __restrict__ Wg, int T, int d,
                                                             int E, int k, int write_routing, int PB,
                                                             float* __restrict__ probs,
                                                             int* __restrict__ idx,
                                                             float* __restrict__ gate, PeerSignal sig) {
  pdl_enter();
  // fused transport: this rank's receive buffers are free again (the previous backward,
  // which read them, is complete in stream order)
  if (blockIdx.x == 0 && threadIdx.x == 0) sig_post(sig);
  constexpr int LP = NT * 8 + 1;
  constexpr int G = NT <= 2 ? 8 : 4;        // 32-column blocks in flight per lane (2 x 16 B each)
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  uint2* frag = reinterpret_cast<uint2*>(gsm_raw);                          // [3][NT][2*PB][32]
  float* part = reinterpret_cast<float*>(gsm_raw + (size_t)3 * NT * 2 * PB * 32 * sizeof(uint2));
  // part: [kGKS][kGTok][LP] partial logits
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int tt = warp % kGTT, kh = warp / kGTT;
  const int t0 = blockIdx.x * kGTok + tt * 16;
  const int ra = t0 + g, rb = t0 + g + 8;
  const bool va = ra < T, vb = rb < T;
  const int nkb = d / 32;
  const int PB2 = 2 * PB;

  float c[NT][4], cm[NT][4], cl[NT][4];  // hi / mid / lo partial products: three independent chains
#pragma unroll
  for (int n = 0; n < NT; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i) c[n][i] = cm[n][i] = cl[n][i] = 0.f;

  for (int p0 = 0; p0 < nkb; p0 += PB) {
    const int pb = min(PB, nkb - p0);
    const int per = (pb + kGKS - 1) / kGKS;
    const int kb0 = p0 + kh * per, kb1 = min(p0 + pb, kb0 + per);
    // first group of this warp's X blocks goes out before the staging
    uint4 xa[G], xb[G];
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const int kb = kb0 + j;
      const int col = kb * 32 + tq * 8;
      const bool in = kb < kb1;
      xa[j] = (in && va) ? *reinterpret_cast<const uint4*>(X + (size_t)ra * d + col) : make_uint4(0, 0, 0, 0);
      xb[j] = (in && vb) ? *reinterpret_cast<const uint4*>(X + (size_t)rb * d + col) : make_uint4(0, 0, 0, 0);
    }
    if (p0) __syncthreads();  // previous pass's fragment reads are done
    // staging: kSB entries per thread per batch, every Wg load of a batch issued before
    // the first split (the loads, not the conversions, are the latency)
    constexpr int kSB = 4;
    const int total = NT * pb * 2 * 32;
    const size_t so = (size_t)NT * PB2 * 32;
    for (int i0 = 0; i0 < total; i0 += kSB * kGThreads) {
      float w[kSB][4];
      int oo[kSB];
#pragma unroll
      for (int u = 0; u < kSB; ++u) {
        const int i = i0 + u * kGThreads + tid;
        const int ln = i & 31, ks = (i >> 5) % (2 * pb), n = (i >> 5) / (2 * pb);
        const int col = (p0 + (ks >> 1)) * 32 + (ln & 3) * 8 + (ks & 1) * 4;
        const int e = n * 8 + (ln >> 2);
        const bool ok = i < total && e < E;
        oo[u] = i < total ? (n * PB2 + ks) * 32 + ln : -1;
#pragma unroll
        for (int q = 0; q < 4; ++q) w[u][q] = ok ? __ldg(Wg + (size_t)(col + q) * E + e) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < kSB; ++u) {
        if (oo[u] < 0) continue;
        float h[4], m[4], l[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) split3(w[u][q], h[q], m[q], l[q]);
        frag[oo[u]] = make_uint2(pack_bf16(h[0], h[1]), pack_bf16(h[2], h[3]));
        frag[so + oo[u]] = make_uint2(pack_bf16(m[0], m[1]), pack_bf16(m[2], m[3]));
        frag[2 * so + oo[u]] = make_uint2(pack_bf16(l[0], l[1]), pack_bf16(l[2], l[3]));
      }
    }
    __syncthreads();
    for (int kbg = kb0; kbg < kb1; kbg += G) {
      if (kbg != kb0) {
#pragma unroll
        for (int j = 0; j < G; ++j) {
          const int kb = kbg + j;
          const int col = kb * 32 + tq * 8;
          const bool in = kb < kb1;
          xa[j] = (in && va) ? *reinterpret_cast<const uint4*>(X + (size_t)ra * d + col) : make_uint4(0, 0, 0, 0);
          xb[j] = (in && vb) ? *reinterpret_cast<const uint4*>(X + (size_t)rb * d + col) : make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int j = 0; j < G; ++j) {
        if (kbg + j >= kb1) break;
        const int kl = kbg + j - p0;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          // logical k (2tq, 2tq+1 | 2tq+8, 2tq+9) <-> physical columns kb*32 + 8tq + 4s + (0,1 | 2,3)
          const uint32_t a[4] = {s ? xa[j].z : xa[j].x, s ? xb[j].z : xb[j].x,
                                 s ? xa[j].w : xa[j].y, s ? xb[j].w : xb[j].y};
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            const size_t o = ((size_t)n * PB2 + 2 * kl + s) * 32 + lane;
            const size_t so = (size_t)NT * PB2 * 32;
            const uint2 bh = frag[o], bm = frag[so + o], bl = frag[2 * so + o];
            mma16816(c[n], a, bh.x, bh.y);
            mma16816(cm[n], a, bm.x, bm.y);
            mma16816(cl[n], a, bl.x, bl.y);
          }
        }
      }
    }
  }
  // fragments -> partial logits: c0,c1 = (row g, cols 2tq, 2tq+1); c2,c3 = (row g+8, ...)
  float* pw = part + (size_t)kh * kGTok * LP;
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    float* r0 = pw + (tt * 16 + g) * LP + n * 8 + 2 * tq;
    float* r1 = pw + (tt * 16 + g + 8) * LP + n * 8 + 2 * tq;
    r0[0] = (c[n][0] + cm[n][0]) + cl[n][0];
    r0[1] = (c[n][1] + cm[n][1]) + cl[n][1];
    r1[0] = (c[n][2] + cm[n][2]) + cl[n][2];
    r1[1] = (c[n][3] + cm[n][3]) + cl[n][3];
  }
  __syncthreads();
  for (int i = tid; i < kGTok * LP; i += kGThreads) {
    float v = part[i];
#pragma unroll
    for (int q = 1; q < kGKS; ++q) v += part[(size_t)q * kGTok * LP + i];
    part[i] = v;
  }
  __syncthreads();
  constexpr int RW = kGTok / (kGThreads / 32);  // logit rows per warp in the epilogue
  gate_epilogue_rows(part + warp * RW * LP, LP, RW, blockIdx.x * kGTok + warp * RW, T, E, k, write_routing,
                     probs, idx, gate);
}

// ------------------------------------------------------------------ SIMT gate (fp32 X)
constexpr int kGateBT = 32;

// EP = padded expert count (8/16/32/64).  Threads: 8 along experts (TE = EP/8 each) x
// 32 along tokens.  DK-column slabs of X (transposed to fp32) and Wg are
// double-buffered through registers.
template <typename TIn, int EP>
__global__ void __launch_bounds__(256) gate_simt_kernel(const TIn* __restrict__ X,
                                                        const float* __restrict__ Wg, int T, int d,
                                                        int E, int k, int write_routing,
                                                        float* __restrict__ probs,
                                                        int* __restrict__ idx,
                                                        float* __restrict__ gate) {
  constexpr int BT = kGateBT;
  constexpr int DK = (EP <= 16) ? 128 : 64;
  constexpr int TE = EP / 8;
  constexpr int XV = BT * DK / 256;
  constexpr int WV = DK * EP / 256;
  __shared__ float xs[DK][BT + 1];
  __shared__ float ws[DK][EP];
  __shared__ float lt[BT][EP + 1];

  const int tid = threadIdx.x;
  const int tx = tid & 7, ty = tid >> 3;
  const int t0 = blockIdx.x * BT;
  constexpr int XT = DK / XV;
  const int xr = tid / XT, xc = (tid % XT) * XV;
  float xreg[XV], wreg[WV];
  auto load_slab = [&](int k0) {
    const int t = t0 + xr;
#pragma unroll
    for (int i = 0; i < XV; i += 8) {
      const int cc = k0 + xc + i;
      if (t < T && cc + 8 <= d && ((d * (int)sizeof(TIn)) % 16 == 0)) {
        const TIn* src = X + (size_t)t * d + cc;
        if constexpr (sizeof(TIn) == 2) {
          load16(src, xreg + i, (const __nv_bfloat16*)nullptr);
        } else {
          load16(src, xreg + i, (const float*)nullptr);
          load16(src + 4, xreg + i + 4, (const float*)nullptr);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          xreg[i + q] = (t < T && cc + q < d) ? Elt<TIn>::to_f(X[(size_t)t * d + cc + q]) : 0.f;
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
    if (k0 + DK < d) load_slab(k0 + DK);  // in flight during the FMAs below
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
  const int warp = tid >> 5;
  gate_epilogue_rows(&lt[warp * 4][0], EP + 1, 4, t0 + warp * 4, T, E, k, write_routing, probs, idx, gate);
}

template <typename TIn, int EP>
void launch_gate_simt(const void* X, const float* Wg, int T, int d, int E, int k, int write_routing,
                      float* probs, int* idx, float* gate, cudaStream_t s) {
  const int blocks = (T + kGateBT - 1) / kGateBT;
  gate_simt_kernel<TIn, EP><<<blocks, 256, 0, s>>>((const TIn*)X, Wg, T, d, E, k, write_routing, probs,
                                                    idx, gate);
}

template <int NT>
void launch_gate_mma(const void* X, const float* Wg, int T, int d, int E, int k, int write_routing,
                     float* probs, int* idx, float* gate, const PeerSignal& sig, cudaStream_t s) {
  const int nkb = d / 32;
  const size_t per_kb = (size_t)3 * NT * 2 * 32 * sizeof(uint2);
  const int PB = (int)std::max<size_t>(1, std::min<size_t>(nkb, kGStageBudget / per_kb));
  const size_t smem = PB * per_kb + sizeof(float) * (size_t)kGKS * kGTok * (NT * 8 + 1);
  static size_t set = 0;
  if (smem > set) {
    LINA_CUDA_CHECK(cudaFuncSetAttribute(gate_mma_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
    set = smem;
  }
  const int blocks = std::max(1, (T + kGTok - 1) / kGTok);  // T = 0: one CTA still posts the signal
  launch_k(gate_mma_kernel<NT>, dim3(blocks), dim3(kGThreads), smem, s, (const __nv_bfloat16*)X, Wg, T, d, E, k,
           write_routing, PB, probs, idx, gate, sig);
}

}  // namespace

void launch_gate_topk(int dtype, const void* X, const float* Wg, int T, int d, int E, int k,
                      int write_routing, float* probs, int* idx, float* gate, cudaStream_t s,
                      const PeerSignal* sig) {
  const PeerSignal none{};
  const PeerSignal& sg = sig ? *sig : none;
  // bf16 tokens: the tcgen05 gate (gate_tc.cu); LINA_GATE_MMA=1 keeps the mma.sync one
  static const bool force_mma = [] {
    const char* e = getenv("LINA_GATE_MMA");
    return e && e[0] == '1';
  }();
  if (dtype == 1 && !force_mma && gate_tc_supported(d, E, k) && (T > 0 || sig)) {
    launch_gate_tc(X, Wg, T, d, E, k, write_routing, probs, idx, gate, sg, s);
    return;
  }
  if (dtype == 1 && d % 32 == 0 && (T > 0 || sig)) {
    const int nt = (E + 7) / 8;
    if (nt <= 1) launch_gate_mma<1>(X, Wg, T, d, E, k, write_routing, probs, idx, gate, sg, s);
    else if (nt <= 2) launch_gate_mma<2>(X, Wg, T, d, E, k, write_routing, probs, idx, gate, sg, s);
    else if (nt <= 4) launch_gate_mma<4>(X, Wg, T, d, E, k, write_routing, probs, idx, gate, sg, s);
    else launch_gate_mma<8>(X, Wg, T, d, E, k, write_routing, probs, idx, gate, sg, s);
  } else {
    if (sig) throw CudaError{"launch_gate_topk: peer signal needs the bf16 tensor-core gate"};
    if (T <= 0) return;
    auto go = [&](auto tag) {
      using TIn = decltype(tag);
      if (E <= 8) launch_gate_simt<TIn, 8>(X, Wg, T, d, E, k, write_routing, probs, idx, gate, s);
      else if (E <= 16) launch_gate_simt<TIn, 16>(X, Wg, T, d, E, k, write_routing, probs, idx, gate, s);
      else if (E <= 32) launch_gate_simt<TIn, 32>(X, Wg, T, d, E, k, write_routing, probs, idx, gate, s);
      else launch_gate_simt<TIn, 64>(X, Wg, T, d, E, k, write_routing, probs, idx, gate, s);
    };
    if (dtype == 0) go(float{});
    else go(__nv_bfloat16{});
  }
  LINA_LAUNCH_CHECK();
}

}  // namespace lina
