// S8 (e)+(f) on the tensor cores: the two gate contractions of the backward,
//   dX_t += Σ_e dL_te · Wg[:, e]      (dx_tc_kernel, fused with the gather-sum of the k
//                                      returned expert input-gradients of token t)
//   dWg   = Σ_t X_tᵀ dL_t              (dwg_tc_kernel, split over tokens, fixed-order reduce)
// with dL_t = p_t ∘ (dp_t − <p_t, dp_t>) (R13; gate_bwd.cu's header).  At C5 (E = 64,
// d = 2048, T = 32768) each is an 8.6 GFLOP contraction that the CUDA-core versions ran
// in 0.5-0.7 ms (profiles/r02_launches_c5_n1.txt); here the tensor cores do the flops and
// the kernels are bound by their HBM reads (X for dWg, the k returned rows for dX).
//
// Precision: dL and Wg are fp32.  Each is split exactly into bf16 terms (x = hi + mid + lo)
// and the products accumulate in fp32 in TMEM:
//   dWg: X is bf16 already, so Xᵀ(dL_hi + dL_mid + dL_lo) is the fp32 product up to order;
//   dX : dL_hi·Wg_hi + dL_hi·Wg_mid + dL_mid·Wg_hi (the dropped terms are < 2^-16 relative),
//        far below the bf16 rounding of the stored dX.
// dl_split_kernel writes dLs [3][T][64] (bf16, E padded to 64 with zeros) once per
// backward; dwg_tc and dx_tc both read it (the workspace region of the dWg partials).
#include <cuda_bf16.h>

#include <algorithm>

#include "../common.h"
#include "../kernels.h"
#include "../signal.h"
#include "tc_ptx.h"

namespace lina {
namespace {

using namespace tc;
constexpr int kEP = 64;  // experts padded (K of dX, N of dWg)

// ---- dL, split: one thread per (token, padded expert)
template <int KM>
__device__ __forceinline__ float token_dot_dp(const float* __restrict__ probs, const int* __restrict__ idx,
                                              const float* __restrict__ gate, const float* __restrict__ dg, int t,
                                              int k, int E, int (&es)[KM], float (&dps)[KM]) {
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
  if (k == 1) {  // g0 = p_e0: dp_e0 = dg0
    dps[0] = dd[0];
#pragma unroll
    for (int j = 1; j < KM; ++j) dps[j] = 0.f;
    return pp[0] * dd[0];
  }
  float S = 0.f, sgd = 0.f;  // g_j = p_ej / S: dp_ei = (dg_i − Σ_j g_j dg_j) / S
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

// one thread per (token, 8 padded experts): the token's <p, dp> once, three 16-byte stores
__global__ void __launch_bounds__(256) dl_split_kernel(const float* __restrict__ probs, const int* __restrict__ idx,
                                                       const float* __restrict__ gate, const float* __restrict__ dg,
                                                       int T, int E, int k, __nv_bfloat16* __restrict__ dls) {
  pdl_enter();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)T * (kEP / 8)) return;
  const int t = (int)(i / (kEP / 8)), e0 = (int)(i % (kEP / 8)) * 8;
  int es[8];
  float dps[8];
  const float dot = token_dot_dp<8>(probs, idx, gate, dg, t, k, E, es, dps);
  __align__(16) __nv_bfloat16 h[8], m[8], l[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = e0 + u;
    float dl = 0.f;
    if (e < E) {
      float dp = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (es[j] == e) dp = dps[j];
      dl = probs[(size_t)t * E + e] * (dp - dot);
    }
    h[u] = __float2bfloat16_rn(dl);
    const float r1 = dl - __bfloat162float(h[u]);
    m[u] = __float2bfloat16_rn(r1);
    l[u] = __float2bfloat16_rn(r1 - __bfloat162float(m[u]));
  }
  const size_t plane = (size_t)T * kEP, o = (size_t)t * kEP + e0;
  *reinterpret_cast<uint4*>(dls + o) = *reinterpret_cast<const uint4*>(h);
  *reinterpret_cast<uint4*>(dls + plane + o) = *reinterpret_cast<const uint4*>(m);
  *reinterpret_cast<uint4*>(dls + 2 * plane + o) = *reinterpret_cast<const uint4*>(l);
}

// WgS [3][d][64]: the terms of Wg[c][e] as rows c (K-major B of the dX contraction)
__global__ void wgt_split_kernel(const float* __restrict__ Wg, int d, int E, __nv_bfloat16* __restrict__ ws) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d * kEP) return;
  const int c = i / kEP, e = i % kEP;
  const float w = e < E ? Wg[(size_t)c * E + e] : 0.f;
  const __nv_bfloat16 hi = __float2bfloat16_rn(w);
  const float r1 = w - __bfloat162float(hi);
  const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
  const __nv_bfloat16 lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
  const size_t plane = (size_t)d * kEP;
  ws[i] = hi;
  ws[plane + i] = mid;
  ws[2 * plane + i] = lo;
}

// ---- dX: a persistent grid; CTA c owns the 256-column block c % nblk of dX (its Wg terms,
// 64 KB, loaded once) and walks the 128-token blocks c / nblk, + G / nblk, ...  Warp 0: TMA
// of the dL terms (3-stage ring); warp 1: 12 MMAs per token block (K = 64 padded experts x
// 3 term pairs) into one of two TMEM accumulators; warps 2..9: the epilogue (thread = token
// row, warps w and w + 4 split the 256 columns), which adds the k returned expert rows and
// stores bf16 dX while the tensor cores work on the next token block — the kernel is bound
// by the epilogue's HBM traffic (read k·d, write d elements per token).
constexpr int kDxA = 128 * kEP * 2;  // 16 KB per dL term
constexpr int kDxB = 256 * kEP * 2;  // 32 KB per Wg term
constexpr int kDxStages = 3;
constexpr int kDxEpw = 8;
constexpr int kDxThreads = 64 + 32 * kDxEpw;
constexpr int kDxSmem = 2 * kDxB + kDxStages * 2 * kDxA + 1024 + 256;

template <int KM>
__global__ void __launch_bounds__(kDxThreads, 1)
    dx_tc_kernel(const __grid_constant__ CUtensorMap tmL, const __grid_constant__ CUtensorMap tmW,
                 const __nv_bfloat16* __restrict__ dXe, const int* __restrict__ idx, const int* __restrict__ slot,
                 int T, int k, int d, int E, int C, int n, int Cm, const int* __restrict__ ebase,
                 __nv_bfloat16* __restrict__ dX, PeerSignal sig) {
  pdl_enter();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sw = smem;                 // Wg hi | Wg mid (resident)
  uint8_t* sl = smem + 2 * kDxB;      // [stage] dL hi | dL mid
  uint64_t* wfull = (uint64_t*)(sl + kDxStages * 2 * kDxA);
  uint64_t* full = wfull + 1;
  uint64_t* empty = full + kDxStages;
  uint64_t* tfull = empty + kDxStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nblk = d / 256;
  const int per = gridDim.x / nblk;  // CTAs per column block (the launcher sizes the grid so)
  const int n0 = (blockIdx.x % nblk) * 256;
  const int tb0 = blockIdx.x / nblk;
  const int ntb = (T + 127) / 128;
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmL);
    prefetch_tmap(&tmW);
    mbar_init(wfull, 1);
    for (int i = 0; i < kDxStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kDxEpw);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc<1>(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // producer and MMA warps walk the token blocks warp-converged; one elected lane issues
  if (warp == 0) {
    if (elect_one()) {
      mbar_expect_tx(wfull, 2 * kDxB);
      tma_load_3d<1>(sw, &tmW, wfull, 0, n0, 0);          // Wg hi
      tma_load_3d<1>(sw + kDxB, &tmW, wfull, 0, n0, 1);   // Wg mid
    }
    __syncwarp();
    int st = 0;
    uint32_t ph = 0;
    for (int tb = tb0; tb < ntb; tb += per) {
      mbar_wait(&empty[st], ph ^ 1);
      uint8_t* dst = sl + st * 2 * kDxA;
      if (elect_one()) {
        mbar_expect_tx(&full[st], 2 * kDxA);
        tma_load_3d<1>(dst, &tmL, &full[st], 0, tb * 128, 0);          // dL hi
        tma_load_3d<1>(dst + kDxA, &tmL, &full[st], 0, tb * 128, 1);   // dL mid
      }
      __syncwarp();
      if (++st == kDxStages) {
        st = 0;
        ph ^= 1;
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16(128, 256, false, false);
    mbar_wait(wfull, 0);
    const uint32_t wa = smem_u32(sw), wm = wa + kDxB;
    const uint64_t wad = sdesc(wa, 16, 1024), wmd = sdesc(wm, 16, 1024);
    int st = 0, acc = 0;
    uint32_t ph = 0, aph = 0;
    for (int tb = tb0; tb < ntb; tb += per) {
      mbar_wait(&tempty[acc], aph ^ 1);
      mbar_wait(&full[st], ph);
      tc_fence_after();
      const uint32_t la = smem_u32(sl + st * 2 * kDxA), lm = la + kDxA;
      const uint64_t lad = sdesc(la, 16, 1024), lmd = sdesc(lm, 16, 1024);
      const uint32_t dt = tmem + acc * 256;
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < kEP / 16; ++kk) {  // +32 B per K = 16 step
          mma_bf16<1>(dt, lad + 2 * kk, wad + 2 * kk, idesc, kk ? 1u : 0u);
          mma_bf16<1>(dt, lad + 2 * kk, wmd + 2 * kk, idesc, 1u);
          mma_bf16<1>(dt, lmd + 2 * kk, wad + 2 * kk, idesc, 1u);
        }
        mma_commit<1>(&empty[st]);
        mma_commit<1>(&tfull[acc]);
      }
      __syncwarp();
      if (++st == kDxStages) {
        st = 0;
        ph ^= 1;
      }
      if (++acc == 2) {
        acc = 0;
        aph ^= 1;
      }
    }
  } else {  // epilogue: thread = token row; + the k returned expert input-gradient rows
    const int ew = warp - 2;
    const int quarter = warp & 3;
    const int c0 = (ew >> 2) * 128;  // this warp's 128 of the block's 256 columns
    if (lane == 0) sig_wait(sig);    // fused transport: the returned rows have landed
    __syncwarp();
    // the k rows' 32-column slices of the next chunk are loaded before the current chunk is
    // summed (two chunks in flight per thread; KM = 2 only — KM = 8 would spill), and the
    // next token block's row indices and first chunk are fetched during the current block's
    // last chunk (no dependent-load bubble between blocks)
    constexpr bool PREF = KM <= 2;
    auto rows_of = [&](int tb, size_t (&rows)[KM]) {
      const int t = tb * 128 + quarter * 32 + lane;
#pragma unroll
      for (int j = 0; j < KM; ++j) {
        rows[j] = ~(size_t)0;
        if (tb < ntb && t < T && j < k) {
          const int s = slot[(size_t)t * k + j];
          const int e = idx[(size_t)t * k + j];
          if (s >= 0) rows[j] = ebase ? (size_t)(ebase[e] + s) : send_row(e, s, E, C, n, Cm);
        }
      }
    };
    auto load_rows = [&](const size_t (&rows)[KM], int cb, uint4 (&dst)[KM][4]) {
#pragma unroll
      for (int j = 0; j < KM; ++j)
#pragma unroll
        for (int v = 0; v < 4; ++v)
          dst[j][v] = rows[j] != ~(size_t)0 ? *reinterpret_cast<const uint4*>(dXe + rows[j] * d + n0 + cb + 8 * v)
                                            : make_uint4(0, 0, 0, 0);
    };
    int acc = 0;
    uint32_t aph = 0;
    uint4 g[PREF ? 2 : 1][KM][4];
    size_t rows[KM];
    rows_of(tb0, rows);
    load_rows(rows, c0, g[0]);
    for (int tb = tb0; tb < ntb; tb += per) {
      const int t = tb * 128 + quarter * 32 + lane;
      size_t nrows[KM];
      if (PREF) rows_of(tb + per, nrows);  // (loads in flight while this block is summed)
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16) + acc * 256;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int cb = c0 + 32 * i;
        float a[32];
        tmem_ld32(ta + cb, *reinterpret_cast<uint32_t(*)[32]>(a));
        if (PREF && i + 1 < 4) load_rows(rows, cb + 32, g[(i + 1) & 1]);
        if (PREF && i == 3) load_rows(nrows, c0, g[0]);  // the next block's first chunk
        if (!PREF && i > 0) load_rows(rows, cb, g[0]);
        uint4 (&cur)[KM][4] = g[PREF ? (i & 1) : 0];
        tmem_wait_ld();
        if (i == 3) {  // the accumulator is read: the MMA warp may reuse it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[acc])) : "memory");
        }
        if (t < T) {
#pragma unroll
          for (int j = 0; j < KM; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              float x[8];
              load16(&cur[j][v], x, (const __nv_bfloat16*)nullptr);
#pragma unroll
              for (int u = 0; u < 8; ++u) a[8 * v + u] += x[u];
            }
#pragma unroll
          for (int v = 0; v < 4; ++v)
            store16(dX + (size_t)t * d + n0 + cb + 8 * v, a + 8 * v, (__nv_bfloat16*)nullptr);
        }
      }
      if (PREF) {
#pragma unroll
        for (int j = 0; j < KM; ++j) rows[j] = nrows[j];
      } else {
        rows_of(tb + per, rows);
        load_rows(rows, c0, g[0]);
      }
      if (++acc == 2) {
        acc = 0;
        aph ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, 512);
  }
  if (sig.bump && threadIdx.x == 0) sig_bump_last(sig);  // the backward's last kernel closes its round
}

// ---- dWg: CTA = 128 columns of d x all 64 (padded) experts, over one token split
constexpr int kDwStages = 4;
constexpr int kDwA = 2 * 64 * 64 * 2;          // X tile: 2 MN blocks of 64 columns x 64 tokens
constexpr int kDwB = 3 * 64 * kEP * 2;         // dL hi / mid / lo: 64 tokens x 64 experts each
constexpr int kDwStage = kDwA + kDwB;
constexpr int kDwSmem = kDwStages * kDwStage + 1024 + 256;

__global__ void __launch_bounds__(192, 1)
    dwg_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmL, int T, int d,
                  int E, int ktok, float* __restrict__ part) {
  pdl_enter();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + kDwStages * kDwStage);
  uint64_t* empty = full + kDwStages;
  uint64_t* tfull = empty + kDwStages;
  uint32_t* tmem_slot = (uint32_t*)(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 128, split = blockIdx.y;
  const int ta = split * ktok, tb = min(T, ta + ktok);
  const int nkb = tb > ta ? (tb - ta + 63) / 64 : 0;
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmL);
    for (int s = 0; s < kDwStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc<1>(tmem_slot, kEP);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // producer and MMA warps walk the K blocks warp-converged; one elected lane issues
  if (warp == 0) {
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      const int t = ta + kb * 64;  // (rows past T are zero-filled by the maps)
      mbar_wait(&empty[stage], ph ^ 1);
      uint8_t* sa = smem + stage * kDwStage;
      if (elect_one()) {
        mbar_expect_tx(&full[stage], kDwStage);
        tma_load_2d<1>(sa, &tmX, &full[stage], m0, t);
        tma_load_2d<1>(sa + 8192, &tmX, &full[stage], m0 + 64, t);
#pragma unroll
        for (int q = 0; q < 3; ++q) tma_load_3d<1>(sa + kDwA + q * 8192, &tmL, &full[stage], 0, t, q);
      }
      __syncwarp();
      if (++stage == kDwStages) {
        stage = 0;
        ph ^= 1;
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16(128, kEP, true, true);  // both operands MN-major
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      mbar_wait(&full[stage], ph);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + stage * kDwStage);
      const uint64_t ad = sdesc(sa, 8192, 1024), bd = sdesc(sa + kDwA, 8192, 1024);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
          for (int q = 0; q < 3; ++q)  // +2 KB per K = 16 step, +8 KB per dL term
            mma_bf16<1>(tmem, ad + 128 * kk, bd + 512 * q + 128 * kk, idesc, (kb | kk | q) ? 1u : 0u);
        mma_commit<1>(&empty[stage]);
      }
      __syncwarp();
      if (++stage == kDwStages) {
        stage = 0;
        ph ^= 1;
      }
    }
    if (elect_one()) mma_commit<1>(tfull);  // (arrives at once when the split is empty)
    __syncwarp();
  } else {
    const int quarter = warp & 3;
    const int c = m0 + quarter * 32 + lane;  // output row = column of d
    mbar_wait(tfull, 0);
    tc_fence_after();
    float acc[kEP];
    const uint32_t tad = tmem + ((uint32_t)(quarter * 32) << 16);
#pragma unroll
    for (int cb = 0; cb < kEP; cb += 32) tmem_ld32(tad + cb, *reinterpret_cast<uint32_t(*)[32]>(acc + cb));
    tmem_wait_ld();
    if (c < d) {
      float* dst = part + ((size_t)split * d + c) * E;
#pragma unroll
      for (int e = 0; e < kEP; ++e)
        if (e < E) dst[e] = nkb ? acc[e] : 0.f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, kEP);
  }
}

// Token splits of dWg: one wave of (d / 128) x S CTAs (one per SM: 160 KB of shared memory
// each) — 2 x 148 / (d / 128) splits ran 2.05 waves at C5 (a third wave of 8 CTAs).
int dwg_tc_splits(int T, int d) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
      sms = 148;
  }
  const int mt = std::max(1, d / 128);
  const int kbs = std::max(1, (T + 63) / 64);
  return std::max(1, std::min(kbs, sms / mt));
}

size_t al256(size_t b) { return (b + 255) / 256 * 256; }

}  // namespace

// As the gate: the tensor-core dX / dWg win once the E-wide contractions dominate (C5:
// 170 + 101 vs 522 + 740 us); at E <= 16 the CUDA-core tiles are faster (C2: 16 + 15 vs
// 28 + 26 us, profiles/r02_launches_c2_n1_*.txt).
bool gate_bwd_tc_supported(int dtype, int d, int E, int k) {
  return dtype == 1 && d % 256 == 0 && E > 16 && E <= kEP && k >= 1 && k <= 8;
}

// Scratch (bytes) of the tensor-core gate backward inside the dWg workspace region:
// partials [S][d][E] fp32 | dLs [3][T][64] bf16 | WgS [3][d][64] bf16.
size_t gate_bwd_tc_scratch_bytes(int T, int d, int E) {
  return al256(sizeof(float) * (size_t)dwg_tc_splits(T, d) * d * E) + al256((size_t)6 * T * kEP) +
         al256((size_t)6 * d * kEP);
}

void launch_dwg_tc(const void* X, const float* probs, const int* idx, const float* gate, const float* dg, int T,
                   int d, int E, int k, void* scratch, float* dWg, cudaStream_t s) {
  const int S = dwg_tc_splits(T, d);
  char* sc = (char*)scratch;
  float* part = (float*)sc;
  __nv_bfloat16* dls = (__nv_bfloat16*)(sc + al256(sizeof(float) * (size_t)S * d * E));
  launch_k(dl_split_kernel, dim3((unsigned)std::max(1LL, ((long long)T * (kEP / 8) + 255) / 256)), dim3(256), 0, s,
           probs, idx, gate, dg, T, E, k, dls);
  LINA_LAUNCH_CHECK();
  const uint64_t xd[2] = {(uint64_t)d, (uint64_t)T};
  const uint64_t xs[1] = {(uint64_t)d * 2};
  const uint32_t xb[2] = {64, 64};
  const CUtensorMap mx = make_map(X, 2, xd, xs, xb);
  const uint64_t ld[3] = {(uint64_t)kEP, (uint64_t)T, 3};
  const uint64_t ls[2] = {(uint64_t)kEP * 2, (uint64_t)T * kEP * 2};
  const uint32_t lb[3] = {(uint32_t)kEP, 64, 1};
  const CUtensorMap ml = make_map(dls, 3, ld, ls, lb);
  static bool attr = false;
  if (!attr) {
    LINA_CUDA_CHECK(cudaFuncSetAttribute(dwg_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDwSmem));
    attr = true;
  }
  const int ktok = ((T + 63) / 64 + S - 1) / S * 64;
  launch_k(dwg_tc_kernel, dim3((d + 127) / 128, S), dim3(192), kDwSmem, s, mx, ml, T, d, E, ktok, part);
  LINA_LAUNCH_CHECK();
  launch_dwg_reduce(part, S, d * E, dWg, s);
}

void launch_dx_tc(const void* dXe, const int* idx, const int* slot, const float* Wg, int T, int k, int d, int E,
                  int C, int n, int Cm, const int* ebase, void* dX, const void* scratch, const PeerSignal& sig,
                  cudaStream_t s) {
  const int S = dwg_tc_splits(T, d);
  const char* sc = (const char*)scratch;
  const __nv_bfloat16* dls = (const __nv_bfloat16*)(sc + al256(sizeof(float) * (size_t)S * d * E));
  __nv_bfloat16* ws = (__nv_bfloat16*)(sc + al256(sizeof(float) * (size_t)S * d * E) + al256((size_t)6 * T * kEP));
  launch_k(wgt_split_kernel, dim3((d * kEP + 255) / 256), dim3(256), 0, s, Wg, d, E, ws);
  LINA_LAUNCH_CHECK();
  const uint64_t ld[3] = {(uint64_t)kEP, (uint64_t)std::max(T, 1), 3};
  const uint64_t ls[2] = {(uint64_t)kEP * 2, (uint64_t)std::max(T, 1) * kEP * 2};
  const uint32_t lb[3] = {(uint32_t)kEP, 128, 1};
  const CUtensorMap ml = make_map(dls, 3, ld, ls, lb);
  const uint64_t wd[3] = {(uint64_t)kEP, (uint64_t)d, 3};
  const uint64_t wsd[2] = {(uint64_t)kEP * 2, (uint64_t)d * kEP * 2};
  const uint32_t wb[3] = {(uint32_t)kEP, 256, 1};
  const CUtensorMap mw = make_map(ws, 3, wd, wsd, wb);
  static bool attr = false;
  if (!attr) {
    LINA_CUDA_CHECK(cudaFuncSetAttribute(dx_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDxSmem));
    LINA_CUDA_CHECK(cudaFuncSetAttribute(dx_tc_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDxSmem));
    attr = true;
  }
  // persistent: a multiple of the column blocks, at most one CTA per SM and per tile
  int dev = 0, sms = 148;
  LINA_CUDA_CHECK(cudaGetDevice(&dev));
  LINA_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int nblk = d / 256, ntb = std::max(1, (T + 127) / 128);
  const int per = std::max(1, std::min(sms / nblk, ntb));
  const dim3 grid(per * nblk);
  if (k <= 2)
    launch_k(dx_tc_kernel<2>, grid, dim3(kDxThreads), kDxSmem, s, ml, mw, (const __nv_bfloat16*)dXe, idx, slot, T, k,
             d, E, C, n, Cm, ebase, (__nv_bfloat16*)dX, sig);
  else
    launch_k(dx_tc_kernel<8>, grid, dim3(kDxThreads), kDxSmem, s, ml, mw, (const __nv_bfloat16*)dXe, idx, slot, T, k,
             d, E, C, n, Cm, ebase, (__nv_bfloat16*)dX, sig);
  LINA_LAUNCH_CHECK();
}

}  // namespace lina
