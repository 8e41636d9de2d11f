// S1 (K1) on the 5th-generation tensor cores: logits X·Wg (tcgen05, fp32 accumulators in
// TMEM) fused with softmax, top-k and the gate weights.
//
// PAPER.md:98 (§2.1): "The gating network takes in the embedding vector of each token and
// multiplies them with its trainable matrix.  Based on the results, it dispatches the
// token to a small number of experts."  Readings R1-R4: softmax over all E
// of X·Wg, no bias; fp32 logits and probabilities; top-k keyed on the logits, ties to the
// lower expert id; k = 1 gate = the raw probability, k >= 2 renormalised over the k.
//
// The contraction is M = T tokens, N = E <= 64 experts, K = d.  The fp32 gate weight is
// split exactly into three bf16 terms (w = hi + mid + lo, 3 x 8 significand bits) once per
// call (gate_split_kernel: Ws [3][EP][d], EP = E padded to 32 or 64 with zero rows), and
// the three products accumulate into ONE TMEM accumulator: per 64-deep K block the CTA
// issues 4 x 3 MMAs (M = 128, N = EP, K = 16) against the same X tile.  Bf16 x bf16
// products are exact in fp32, so the logits equal the fp32 contraction up to accumulation
// order — exact for the grid inputs of DESIGN.md §4.
//
// One CTA per 128 tokens, warp-specialised: warp 0 = TMA producer (X tile 128 x 64 and the
// three Ws slabs EP x 64, 128B-swizzled, 2-stage ring, two CTAs per SM), warp 1 = TMEM allocator + MMA
// issuer, warps 2..5 = epilogue: tcgen05.ld puts one token's EP logits in one thread's
// registers, which computes the softmax, the top-k and the gate weights without any
// shuffle and stores its probabilities row (16-byte stores).  X is read once: the kernel
// is bound by that read (C5: 134 MB), where the mma.sync version it replaces re-staged the
// split Wg per 32 tokens (profiles/r02_launches_c5_n1.txt: 377 us at C5).
#include <cuda_bf16.h>
#include <math.h>

#include <map>
#include <mutex>
#include <tuple>

#include "../common.h"
#include "../kernels.h"
#include "../signal.h"
#include "tc_ptx.h"

namespace lina {
namespace {

using namespace tc;

constexpr int kGBK = 64;       // K per stage: 128-byte rows, one swizzle atom wide
// 2 stages (<= 81 KB of shared memory): two CTAs per SM, so C5's 256 token blocks run in one
// wave (4 stages, one CTA per SM: 1.73 waves) and one CTA's epilogue overlaps the other's loads
constexpr int kGStages = 2;
constexpr int kGThreads = 192;  // warp 0 TMA, warp 1 MMA, warps 2..5 epilogue

template <int EP>
struct GGeo {
  static constexpr int A_BYTES = 128 * kGBK * 2;     // 16 KB X tile
  static constexpr int B_BYTES = 3 * EP * kGBK * 2;  // hi / mid / lo slabs
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int SMEM = kGStages * STAGE + 1024 /*align*/ + 256 /*barriers*/;
};

// Ws[q][e][c] = term q of Wg[c][e] (q = 0 hi, 1 mid, 2 lo); rows e >= E are zero.
__global__ void gate_split_kernel(const float* __restrict__ Wg, int d, int E, int EP,
                                  __nv_bfloat16* __restrict__ Ws) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d * EP) return;
  const int e = i / d, c = i % d;
  const float w = e < E ? Wg[(size_t)c * E + e] : 0.f;
  const __nv_bfloat16 hi = __float2bfloat16_rn(w);
  const float r1 = w - __bfloat162float(hi);
  const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
  const __nv_bfloat16 lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));  // exact: <= 8 bits left
  Ws[((size_t)0 * EP + e) * d + c] = hi;
  Ws[((size_t)1 * EP + e) * d + c] = mid;
  Ws[((size_t)2 * EP + e) * d + c] = lo;
}

template <int EP>
__global__ void __launch_bounds__(kGThreads, 2)
    gate_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, int T, int d,
                   int E, int k, int write_routing, float* __restrict__ probs, int* __restrict__ idx,
                   float* __restrict__ gate, PeerSignal sig) {
  using G = GGeo<EP>;
  pdl_enter();
  // fused transport: this rank's receive buffers of the round are free (block 0 posts)
  if (blockIdx.x == 0 && threadIdx.x == 0) sig_post(sig);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + kGStages * G::STAGE);
  uint64_t* empty = full + kGStages;
  uint64_t* tfull = empty + kGStages;
  uint32_t* tmem_slot = (uint32_t*)(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 128;
  const int nkb = d / kGBK;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmW);
    for (int s = 0; s < kGStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc<1>(tmem_slot, EP);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // producer and MMA warps walk the K blocks warp-converged (operands in uniform registers);
  // one elected lane issues the loads / MMAs
  if (warp == 0) {  // ---- TMA producer
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      mbar_wait(&empty[stage], ph ^ 1);
      uint8_t* sa = smem + stage * G::STAGE;
      if (elect_one()) {
        mbar_expect_tx(&full[stage], G::STAGE);
        tma_load_2d<1>(sa, &tmX, &full[stage], kb * kGBK, m0);
        tma_load_2d<1>(sa + G::A_BYTES, &tmW, &full[stage], kb * kGBK, 0);
      }
      __syncwarp();
      if (++stage == kGStages) {
        stage = 0;
        ph ^= 1;
      }
    }
  } else if (warp == 1) {  // ---- MMA issuer: hi, mid and lo products into one accumulator
    constexpr uint32_t idesc = idesc_bf16(128, EP, false, false);
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      mbar_wait(&full[stage], ph);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + stage * G::STAGE);
      const uint64_t ad = sdesc(sa, 16, 1024), bd = sdesc(sa + G::A_BYTES, 16, 1024);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < kGBK / 16; ++kk)
#pragma unroll
          for (int q = 0; q < 3; ++q)  // +32 B per K = 16 step, +EP rows x 128 B per term
            mma_bf16<1>(tmem, ad + 2 * kk, bd + 2 * kk + q * EP * 8, idesc, (kb | kk | q) ? 1u : 0u);
        mma_commit<1>(&empty[stage]);
      }
      __syncwarp();
      if (++stage == kGStages) {
        stage = 0;
        ph ^= 1;
      }
    }
    if (elect_one()) mma_commit<1>(tfull);
    __syncwarp();
  } else {  // ---- epilogue: one token per thread
    const int quarter = warp & 3;
    const int t = m0 + quarter * 32 + lane;
    mbar_wait(tfull, 0);
    tc_fence_after();
    float l[EP];
    const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16);
#pragma unroll
    for (int c = 0; c < EP; c += 32) tmem_ld32(ta + c, *reinterpret_cast<uint32_t(*)[32]>(l + c));
    tmem_wait_ld();
    if (t < T) {
      float mx = -INFINITY;
#pragma unroll
      for (int e = 0; e < EP; ++e)
        if (e < E) mx = fmaxf(mx, l[e]);
      float z[EP];
      float sum = 0.f;
#pragma unroll
      for (int e = 0; e < EP; ++e) {
        z[e] = e < E ? expf(l[e] - mx) : 0.f;
        sum += z[e];
      }
#pragma unroll
      for (int e = 0; e < EP; ++e) z[e] = z[e] / sum;  // probabilities
      float* prow = probs + (size_t)t * E;
      if ((E & 3) == 0) {
#pragma unroll
        for (int e = 0; e < EP; e += 4)
          if (e < E) *reinterpret_cast<float4*>(prow + e) = make_float4(z[e], z[e + 1], z[e + 2], z[e + 3]);
      } else {
#pragma unroll
        for (int e = 0; e < EP; ++e)
          if (e < E) prow[e] = z[e];
      }
      if (write_routing) {
        uint64_t taken = 0;
        float ps[8];
        float psum = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j >= k) break;
          float bl = -INFINITY, bp = 0.f;
          int bi = -1;
#pragma unroll
          for (int e = 0; e < EP; ++e)  // ascending e: a tie keeps the lower id (R3)
            if (e < E && !((taken >> e) & 1ull) && (bi < 0 || l[e] > bl)) {
              bl = l[e];
              bi = e;
              bp = z[e];
            }
          taken |= 1ull << bi;
          idx[(size_t)t * k + j] = bi;
          ps[j] = bp;
          psum += bp;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j < k) gate[(size_t)t * k + j] = k == 1 ? ps[0] : ps[j] / psum;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, EP);
  }
}

// The split weights live in a device buffer per (device, d, EP), allocated by the first
// (eager) call; every call rewrites it from the current Wg.
__nv_bfloat16* split_buffer(int d, int EP) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int>, __nv_bfloat16*> bufs;
  int dev = 0;
  LINA_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  auto key = std::make_tuple(dev, d, EP);
  auto it = bufs.find(key);
  if (it != bufs.end()) return it->second;
  __nv_bfloat16* p = nullptr;
  LINA_CUDA_CHECK(cudaMalloc(&p, sizeof(__nv_bfloat16) * 3 * (size_t)EP * d));
  bufs[key] = p;
  return p;
}

template <int EP>
void launch_gate_tc_t(const void* X, const float* Wg, int T, int d, int E, int k, int write_routing, float* probs,
                      int* idx, float* gate, const PeerSignal& sig, cudaStream_t s) {
  __nv_bfloat16* ws = split_buffer(d, EP);
  launch_k(gate_split_kernel, dim3((d * EP + 255) / 256), dim3(256), 0, s, Wg, d, E, EP, ws);
  LINA_LAUNCH_CHECK();
  const uint64_t xd[2] = {(uint64_t)d, (uint64_t)std::max(T, 1)};
  const uint64_t xs[1] = {(uint64_t)d * 2};
  const uint32_t xb[2] = {kGBK, 128};
  const CUtensorMap mx = make_map(X, 2, xd, xs, xb);
  const uint64_t wd[2] = {(uint64_t)d, (uint64_t)3 * EP};
  const uint64_t wsd[1] = {(uint64_t)d * 2};
  const uint32_t wb[2] = {kGBK, (uint32_t)(3 * EP)};
  const CUtensorMap mw = make_map(ws, 2, wd, wsd, wb);
  static bool attr = false;
  if (!attr) {
    LINA_CUDA_CHECK(
        cudaFuncSetAttribute(gate_tc_kernel<EP>, cudaFuncAttributeMaxDynamicSharedMemorySize, GGeo<EP>::SMEM));
    attr = true;
  }
  const int blocks = std::max(1, (T + 127) / 128);  // T = 0: one CTA still posts the signal
  launch_k(gate_tc_kernel<EP>, dim3(blocks), dim3(kGThreads), GGeo<EP>::SMEM, s, mx, mw, T, d, E, k, write_routing,
           probs, idx, gate, sig);
}

}  // namespace

// The tensor-core gate pays off once E is large (C5, E = 64: 60 vs 377 us); for E <= 16 the
// mma.sync kernel's staged split Wg is small and its 32-token CTAs fill the GPU at small T
// (C2, E = 8, T = 8192: 10.9 vs 18 + 3 us, profiles/r02_launches_c2_n1_*.txt).
bool gate_tc_supported(int d, int E, int k) { return d % kGBK == 0 && d > 0 && E > 16 && E <= 64 && k <= 8; }

void launch_gate_tc(const void* X, const float* Wg, int T, int d, int E, int k, int write_routing, float* probs,
                    int* idx, float* gate, const PeerSignal& sig, cudaStream_t s) {
  if (E <= 32) launch_gate_tc_t<32>(X, Wg, T, d, E, k, write_routing, probs, idx, gate, sig, s);
  else launch_gate_tc_t<64>(X, Wg, T, d, E, k, write_routing, probs, idx, gate, sig, s);
  LINA_LAUNCH_CHECK();
}

}  // namespace lina
