// S5 / S8c expert FFN GEMMs on the 5th-generation tensor cores (bf16 in, fp32 accumulate).
//
// "Every expert is a fully-connected two-layer network using ReLU"; the
// expert GEMMs are the only dense contraction on the path.
//
// One persistent, warp-specialised kernel per (CTA-group, problem, B-major, epilogue):
//   warp 0      : TMA producer (one elected lane issues) — A and B tiles into a
//                 128B-swizzled shared-memory ring, completion on mbarriers;
//   warp 1      : TMEM allocator + MMA issuer (one elected lane of the leader CTA issues) —
//                 tcgen05.mma.kind::f16, K=16 per instruction, fp32 accumulators
//                 in TMEM, double-buffered (2 x 256 columns) so the epilogue of
//                 tile i overlaps the MMAs of tile i+1;
//   warps 2..5  : epilogue — tcgen05.ld 32x32b (one TMEM lane = one row per
//                 thread), ReLU / ReLU'-mask, bf16 rounding, 16-byte stores.
// CG = 2 (default): a CTA pair (cluster 2x1) computes a 256 x 256 tile with
//   tcgen05.mma.cta_group::2 (UMMA M=256): each CTA stages its 128 rows of A and
//   its half (128 columns) of B, so every SM streams 32 KB per 64-deep K block
//   instead of 48 KB — the L2->SM feed, not the tensor pipe, bounded the 1-CTA
//   version at ~66% tensor activity (profiles/r01_*).  TMA completions of both CTAs
//   land on the leader's mbarrier; MMA completion is multicast to both CTAs.
// CG = 1: single-CTA M=128 N=256 (kept for shapes whose row count is small).
// Two problem shapes share the kernel:
//   ROW   (forward GEMM1/GEMM2, backward dgrad): D[seg rows] = epi(A[seg rows] · B_eᵀ)
//         over the (segment, row-block) tiles that hold valid rows, A viewed by a
//         3-D tensor map [segments][Cm rows][K] so a tile never reads past its
//         segment (TMA zero-fills); B_e K-major (W as stored) or MN-major (the
//         transposed use of the other weight in dgrad).
//   WGRAD (backward weight gradients): D_e[M][N] = Σ_segments Σ_rows A_rᵀ B_r with
//         both operands MN-major views of row buffers; the K loop walks the valid
//         rows of every (chunk, source) segment of expert e in 64-row blocks.
// Tiles are handed out over a grid of #SMs CTAs, statically per cluster or (long K / many
// waves) dynamically from a per-communicator ticket counter (TcParams::tile_ctr); ROW tiles
// are enumerated from a per-chunk prefix of valid row blocks (launch_mtile_prefix).  The
// producer and MMA warps run warp-converged and issue from one elect.sync lane.
#include <cuda.h>

#include <stdlib.h>

#include <cstring>

#include "../common.h"
#include "../kernels.h"
#include "../signal.h"
#include "tc_ptx.h"

namespace lina {
namespace tc {

constexpr int BN = 256, BK = 64;
constexpr int TMEM_COLS = 512;  // 2 accumulators x BN

// WIDE: the epilogue-heavy ReLU / ReLU'-mask GEMMs (N = d_ffn outputs per row, short
// K = d_model) get 8 epilogue warps (two per TMEM lane quarter, each owning half of
// the 256 columns).  WIDE = 1 gives up one pipeline stage for their double-buffered
// staging boxes; WIDE = 2 keeps every stage and single-buffers the boxes (a warp waits
// for its previous box's TMA store to have read the buffer before refilling it).
template <int CG, int WIDE = 0> struct Geo {
  static constexpr int ROWS = 128 * CG;                  // tile rows per cluster
  static constexpr int A_BYTES = 128 * BK * 2;           // 16 KB per CTA
  static constexpr int B_ROWS = BN / CG;                 // B rows (N) staged per CTA
  static constexpr int B_BYTES = B_ROWS * BK * 2;        // 32 KB (CG=1) / 16 KB (CG=2)
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (CG == 2 ? 6 : 4) - (WIDE == 1 ? 1 : 0);
  static constexpr int EPW = WIDE ? 8 : 4;               // epilogue warps
  static constexpr int THREADS = 64 + 32 * EPW;
  static constexpr int EPI_BUFS = WIDE == 2 ? 1 : 2;     // 32 rows x 128 B boxes per epilogue warp
  static constexpr int EPI_BYTES = EPW * EPI_BUFS * 4096;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*align*/ + 512 /*barriers*/;
};

constexpr int kMaxPeerMaps = 8;

struct TcParams {
  const int* vcount;   // valid rows per segment (global segment index)
  const int* mtp;      // ROW: [nseg+1] prefix of valid row blocks of this launch's segments
  const int* seg_expert;  // ROW: weight index of local slot (seg % El); NULL = identity
  int seg0, nseg, El, Cm;
  int M, N, K;         // WGRAD: M x N output per expert; ROW: N, K
  __nv_bfloat16* D;
  const __nv_bfloat16* aux;
  int nchunks, P;      // WGRAD
  const int* seg_range;  // WGRAD, dropless layout: expert el's segments [seg_range[2el], seg_range[2el+1])
  const int* row_base;   // ROW tail launches: first row of each (global) segment's tail tile
  // ROW with peer stores: output tile of segment (c, s, el) goes through pmaps[s] to
  // segment c*dE + dme*El + el of rank s's buffer (the combine all-to-all fused into
  // the epilogue); has_pmaps = 0: local store through tmD
  int has_pmaps;
  int dP, dme, dE;
  uint64_t* mask_out;       // ROW + ReLU: ReLU' bits of the stored output, [seg][N/64][Cm]
  const uint64_t* mask_in;  // ROW + mask epilogue: the bits written by GEMM1
  PeerSignal sig;           // fused transport: wait before the first A load / post after the last store
  int src_wait;             // ROW: sig.wait per source (segment (c, s, el) waits for s only), tiles from dme up
  CUtensorMap pmaps[kMaxPeerMaps];  // kernel-parameter copies (the TMA unit reads them like tmD)
  char* pbase[kMaxPeerMaps];        // the same buffers as plain pointers (remote owners: SM stores)
  // ROW, CG = 2: a segment's last m-tile holding <= 128 valid rows runs as an M = 128
  // cta_group::2 tile (64 rows per CTA, loaded through tmA64) — half the MMA time of the
  // M = 256 tile it would otherwise pad to.  Accumulator: the 2x2 data-path layout (per
  // CTA, columns [0, 128) in TMEM lanes 0-63 and [128, 256) in lanes 64-127, 128 columns).
  int half;
  CUtensorMap tmA64;
  // Dynamic tile schedule (NULL: static, cluster c takes tiles c, c + #clusters, ...): the
  // leader CTA's producer takes the next tile from this counter and hands it to its MMA and
  // epilogue warps and to the peer CTA through a 4-deep shared-memory queue, so the tiles in
  // flight stay a contiguous window whatever their lengths (half tails, unequal wgrad K) and
  // the clusters reuse each other's operands from L2.  The cluster drawing the last ticket
  // (#tiles + #clusters - 1) resets the counter to 0 for the next launch (stream order).
  unsigned int* tile_ctr;
  int dyn_static;  // A/B only (LINA_GEMM_DYN=3): the queue hand-off with the static tile order
};

constexpr int kQ = 4;  // tile-queue depth

template <int CG, bool WGRAD, bool B_MN, int EPI, int WIDE = (EPI != kEpiNone)>
__global__ void __launch_bounds__(Geo<CG, WIDE>::THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmX,
                   const __grid_constant__ TcParams p) {
  pdl_enter();
  using G = Geo<CG, WIDE>;
  constexpr int STAGES = G::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* epi_smem = smem + STAGES * G::STAGE_BYTES;   // [4 warps][2 buffers][32 rows][128 B]
  uint64_t* full = (uint64_t*)(epi_smem + G::EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_base_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr bool A_MN = WGRAD;  // wgrad: A = (dO or dH) rows viewed MN-major
  const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x / CG, num_clusters = gridDim.x / CG;

  // ---- tile space (per cluster)
  const int n_nblk = p.N / BN;
  const int total_tiles = WGRAD ? p.El * (p.M / G::ROWS) * n_nblk : p.mtp[p.nseg] * n_nblk;
  const bool dyn = p.tile_ctr != nullptr;
  if (!dyn && cluster_id >= total_tiles) {  // uniform for the whole cluster
    if (threadIdx.x == 0) sig_post_last(p.sig);  // still counts towards the grid's completion
    return;
  }

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    prefetch_tmap(&tmD);
    if (EPI == kEpiMask) prefetch_tmap(&tmX);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], G::EPW * CG);
    }
    for (int a = 0; a < 16; ++a) mbar_init(tempty + 3 + a, 1);  // epilogue aux-box barriers
    for (int a = 0; a < kQ; ++a) {  // tile queue: one producer; leader MMA + producer of the peer + all epilogue warps
      mbar_init(tempty + 19 + a, 1);
      mbar_init(tempty + 19 + kQ + a, (CG == 2 ? 2 : 1) + CG * G::EPW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc<CG>(tmem_base_slot, TMEM_COLS);
  tc_fence_before();
  if (CG == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  uint64_t* qfull = tempty + 19;
  uint64_t* qempty = qfull + kQ;
  volatile int* tq = (volatile int*)(qempty + kQ);
  // Tile queue of the dynamic schedule.  Leader producer: publish ticket t (drawn a tile
  // earlier, its atomic in flight during that tile's loads) to the queue of both CTAs
  auto q_publish = [&](int& qi, uint32_t& qph, int t) {
    mbar_wait(&qempty[qi], qph ^ 1);  // (acquire.cta: an acquire.cluster wait would invalidate L1)
    if (lane == 0) {
      tq[qi] = t;
      mbar_arrive_local(&qfull[qi]);
      if (CG == 2) st_async_cluster_s32((const void*)&tq[qi], &qfull[qi], 1, t);
      if (!p.dyn_static && t == total_tiles + num_clusters - 1) atomicExch(p.tile_ctr, 0u);  // the last ticket
    }
    t = __shfl_sync(0xffffffffu, t, 0);
    if (++qi == kQ) {
      qi = 0;
      qph ^= 1;
    }
    return t;
  };
  int n_draw = 0;
  auto q_draw = [&]() {
    const int i = n_draw++;
    if (p.dyn_static) return cluster_id + i * num_clusters;
    return lane == 0 ? (int)atomicAdd(p.tile_ctr, 1u) : 0;
  };
  // consumers; in the peer CTA its producer registers the 4 bytes of each ticket's st.async
  // (with that phase's arrival), the other consumers only wait
  auto q_take = [&](int& qi, uint32_t& qph) {
    if (rank != 0 && warp == 0 && lane == 0) mbar_expect_tx(&qfull[qi], 4);
    mbar_wait(&qfull[qi], qph);
    const int t = tq[qi];
    __syncwarp();
    if (lane == 0) {
      if (rank == 0) mbar_arrive_local(&qempty[qi]);
      else mbar_arrive_cluster_relaxed(&qempty[qi], 0);
    }
    if (++qi == kQ) {
      qi = 0;
      qph ^= 1;
    }
    return t;
  };
  auto next_tile = [&](int it, int& qi, uint32_t& qph) {
    return dyn ? q_take(qi, qph) : cluster_id + it * num_clusters;
  };

  // Fused combine stores: every rank starts at the tiles of source (me + 1) % P, so at any
  // moment the P ranks write to P different owners (no incast on one rank's links).
  // Split dispatch (src_wait): start at this rank's own source, whose rows are local, then
  // me + 1, me + 2, ... — the order the peers' rows arrive in (permute.cu split_rows_kernel).
  const int rot = (!WGRAD && p.has_pmaps && p.dP > 1) ? p.mtp[((p.dme + 1) % p.dP) * p.El] * n_nblk
                  : (!WGRAD && p.src_wait && p.dP > 1) ? p.mtp[p.dme * p.El] * n_nblk
                                                       : 0;
  auto decode = [&](int t0, int& seg_or_el, int& m0, int& n0) {
    int t = t0 + rot;
    if (t >= total_tiles) t -= total_tiles;
    const int nb = t % n_nblk;
    const int ml = t / n_nblk;
    n0 = nb * BN;
    if (WGRAD) {
      const int mblks = p.M / G::ROWS;
      seg_or_el = ml / mblks;
      m0 = (ml % mblks) * G::ROWS;
    } else {
      // the last segment whose first m-tile is <= ml (binary search over the prefix; an
      // empty segment shares its start with the next one, so the last such is non-empty)
      int i = 0, hi = p.nseg - 1;
      while (i < hi) {
        const int mid = (i + hi + 1) >> 1;
        if (__ldg(p.mtp + mid) <= ml) i = mid;
        else hi = mid - 1;
      }
      seg_or_el = i;  // local segment index within this launch
      m0 = (ml - p.mtp[i]) * G::ROWS + (p.row_base ? __ldg(p.row_base + p.seg0 + i) : 0);
    }
  };
  // ROW, CG = 2: does the tile at (local segment se, first row m0) hold <= 128 valid rows?
  auto half_of = [&](int se, int m0) {
    return CG == 2 && !WGRAD && p.half && __ldg(p.vcount + p.seg0 + se) - m0 <= 128;
  };
  auto kblocks_of = [&](int seg_or_el) {
    if (!WGRAD) return p.K / BK;
    int kb = 0;
    if (p.seg_range) {
      for (int seg = p.seg_range[2 * seg_or_el]; seg < p.seg_range[2 * seg_or_el + 1]; ++seg)
        kb += (p.vcount[seg] + BK - 1) / BK;
      return kb;
    }
    for (int c = 0; c < p.nchunks; ++c)
      for (int s = 0; s < p.P; ++s) kb += (p.vcount[(c * p.P + s) * p.El + seg_or_el] + BK - 1) / BK;
    return kb;
  };

  if (warp == 0) {
    // ================= TMA producer (both CTAs load their own halves): the whole warp walks
    // the tiles and waits (warp-uniform, operands in uniform registers); one elected lane
    // issues the loads
    {
      if (p.sig.wait && !p.src_wait) {  // fused transport: the peers' rows of A have landed
        if (elect_one()) {
          sig_wait(p.sig);
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        __syncwarp();
      }
      uint32_t have = 1u << p.dme;  // split dispatch: sources whose rows are known to be in
      int stage = 0;
      uint32_t ph = 0;
      const int arow = 128 * rank;          // this CTA's rows within the tile
      const int brow = G::B_ROWS * rank;    // this CTA's B (N) rows within the tile
      int qi = 0;
      uint32_t qph = 0;
      // dynamic schedule, leader: the next tile's ticket is drawn when this tile starts and
      // published when its loads are issued (the atomic's latency hides behind them)
      int t_next = dyn && leader ? q_publish(qi, qph, q_draw()) : 0;
      for (int it = 0;; ++it) {
        const int t = !dyn ? cluster_id + it * num_clusters : leader ? t_next : q_take(qi, qph);
        if (t >= total_tiles) break;
        const int drawn = dyn && leader ? q_draw() : 0;
        int se, m0, n0;
        decode(t, se, m0, n0);
        const bool hf = !WGRAD && half_of(se, m0);
        auto issue = [&](int a0, int a1, int a2, int b0, int b1, int b2) {
          mbar_wait(&empty[stage], ph ^ 1);
          uint8_t* sa = smem + stage * G::STAGE_BYTES;
          uint8_t* sb = sa + G::A_BYTES;
          if (elect_one()) {
          if (leader) mbar_expect_tx(&full[stage], CG * (hf ? G::STAGE_BYTES - G::A_BYTES / 2 : G::STAGE_BYTES));
          if (!A_MN && hf) {
            tma_load_3d<CG>(sa, &p.tmA64, &full[stage], a0, a1 - 64 * (int)rank, a2);  // rows m0 + 64 * rank
          } else if (!A_MN) {
            tma_load_3d<CG>(sa, &tmA, &full[stage], a0, a1, a2);
          } else {
#pragma unroll
            for (int j = 0; j < 2; ++j) tma_load_3d<CG>(sa + j * 8192, &tmA, &full[stage], a0 + j * 64, a1, a2);
          }
          if (!B_MN) {
            tma_load_2d<CG>(sb, &tmB, &full[stage], b0, b1);
          } else if (!WGRAD) {
#pragma unroll
            for (int j = 0; j < G::B_ROWS / 64; ++j)
              tma_load_2d<CG>(sb + j * 8192, &tmB, &full[stage], b0 + j * 64, b1);
          } else {
#pragma unroll
            for (int j = 0; j < G::B_ROWS / 64; ++j)
              tma_load_3d<CG>(sb + j * 8192, &tmB, &full[stage], b0 + j * 64, b1, b2);
          }
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            ph ^= 1;
          }
        };
        if (!WGRAD) {
          const int seg = p.seg0 + se;
          if (p.src_wait) {
            const int src = (seg / p.El) % p.dP;
            if (!((have >> src) & 1u)) {
              if (elect_one()) {
                sig_wait_one(p.sig, src);
                asm volatile("fence.proxy.async.global;" ::: "memory");
              }
              __syncwarp();
              have |= 1u << src;
            }
          }
          const int el = p.seg_expert ? p.seg_expert[se % p.El] : se % p.El;
          for (int kb = 0; kb < p.K / BK; ++kb) {
            const int k0 = kb * BK;
            if (!B_MN) issue(k0, m0 + arow, seg, k0, el * p.N + n0 + brow, 0);
            else issue(k0, m0 + arow, seg, n0 + brow, el * p.K + k0, 0);
          }
        } else {
          const int el = se;
          if (p.seg_range) {
            for (int seg = p.seg_range[2 * el]; seg < p.seg_range[2 * el + 1]; ++seg) {
              const int v = p.vcount[seg];
              for (int r0 = 0; r0 < v; r0 += BK) issue(m0 + arow, r0, seg, n0 + brow, r0, seg);
            }
          } else {
            for (int c = 0; c < p.nchunks; ++c)
              for (int s = 0; s < p.P; ++s) {
                const int seg = (c * p.P + s) * p.El + el;
                const int v = p.vcount[seg];
                for (int r0 = 0; r0 < v; r0 += BK) issue(m0 + arow, r0, seg, n0 + brow, r0, seg);
              }
          }
        }
        if (dyn && leader) t_next = q_publish(qi, qph, drawn);
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (leader CTA only): the whole warp walks the tiles and
    // waits (warp-uniform control flow, operands in uniform registers); one elected lane
    // issues the MMAs and commits.  Per 64-deep K block the stage's descriptors are built
    // once and advanced per K = 16 step by a constant (+32 B K-major, +2 KB MN-major).
    if (leader) {
      constexpr uint32_t idesc_full = idesc_bf16(G::ROWS, BN, A_MN, B_MN);
      constexpr uint32_t idesc_half = idesc_bf16(128, BN, A_MN, B_MN);
      constexpr uint64_t a_step = A_MN ? 2048 >> 4 : 32 >> 4, b_step = B_MN ? 2048 >> 4 : 32 >> 4;
      const uint32_t smem0 = smem_u32(smem);
      int stage = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      int qi = 0;
      uint32_t qph = 0;
      for (int it = 0;; ++it) {
        const int t = next_tile(it, qi, qph);
        if (t >= total_tiles) break;
        int se, m0, n0;
        decode(t, se, m0, n0);
        const int nkb = kblocks_of(se);
        const uint32_t idesc = half_of(se, m0) ? idesc_half : idesc_full;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], ph);
          tc_fence_after();
          const uint32_t sa = smem0 + stage * G::STAGE_BYTES;
          const uint32_t sb = sa + G::A_BYTES;
          // K-major SW128: +32 B per K=16 step inside the 128 B atom; SBO = 8 rows * 128 B.
          // MN-major SW128: +2 x (8 K-rows * 128 B) per K=16 step; LBO = 64-element MN block.
          const uint64_t ad = A_MN ? sdesc(sa, 8192, 1024) : sdesc(sa, 16, 1024);
          const uint64_t bd = B_MN ? sdesc(sb, 8192, 1024) : sdesc(sb, 16, 1024);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              mma_bf16<CG>(d_tmem, ad + a_step * kk, bd + b_step * kk, idesc, (kb | kk) ? 1u : 0u);
            mma_commit<CG>(&empty[stage]);  // frees the smem slot (in both CTAs) once read
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            ph ^= 1;
          }
        }
        if (elect_one()) mma_commit<CG>(&tfull[acc]);  // accumulator ready (arrives at once if nkb == 0)
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          aph ^= 1;
        }
      }
    }
  } else {
    // ================= epilogue (warps 2..): TMEM lane quarter = warp % 4
    // Each warp owns 32 rows and BN/(EPW/4) columns: TMEM -> registers -> epi -> bf16 ->
    // a 128B-swizzled 32 x 64 smem box -> TMA store (rows past the segment end are
    // clipped by the tensor map).  Two boxes per warp alternate so the store of one
    // overlaps the fill of the next.  The ReLU epilogue (GEMM1) also emits the ReLU'
    // bits of the bf16 H it stores (one 64-bit word per row and 64 columns); the dgrad
    // epilogue multiplies by those bits instead of re-reading H (6 MB instead of 100 MB
    // at configs[1]).
    const int ew = warp - 2;                 // epilogue warp index
    const int quarter = warp & 3;
    constexpr int COLS = BN / (G::EPW / 4);  // columns per warp
    uint8_t* my_epi = epi_smem + ew * G::EPI_BUFS * 4096;
    int acc = 0;
    uint32_t aph = 0;
    int sub = 0;  // sub-tile counter (buffer = sub & 1)
    const int mwords = p.N >> 6;
    int qi = 0;
    uint32_t qph = 0;
    for (int it = 0;; ++it) {
      const int t = next_tile(it, qi, qph);
      if (t >= total_tiles) break;
      int se, m0, n0;
      decode(t, se, m0, n0);
      const int nkb = kblocks_of(se);
      // full tile: this warp's 32 rows = TMEM lanes of its quarter, COLS columns from col0;
      // half tile (2x2 layout): quarters 0/1 hold rows 0-31 / 32-63 of this CTA's 64 rows
      // with output columns [0, 128), quarters 2/3 the same rows with columns [128, 256), all
      // in TMEM columns [0, 128) — COLS / 2 columns per warp
      const bool hf = half_of(se, m0);
      const int rbase = hf ? m0 + 64 * rank + (quarter & 1) * 32 : m0 + 128 * rank + quarter * 32;
      const int col0 = hf ? (quarter >> 1) * 128 + (ew >> 2) * (COLS / 2) : (ew >> 2) * COLS;  // output column
      const int tcol0 = hf ? (ew >> 2) * (COLS / 2) : col0;                                   // TMEM column
      const int njs = hf ? COLS / 128 : COLS / 64;  // 64-column boxes of this warp
      const int row = rbase + lane;  // row within the segment
      const bool row_ok = !WGRAD && row < p.Cm;
      // ReLU' words are word-column-major, [seg][N/64][Cm]: the 32 lanes (32 consecutive
      // rows) of a warp store / load 256 contiguous bytes per word column
      const size_t mrow = row_ok ? ((size_t)(p.seg0 + se) * mwords + ((n0 + col0) >> 6)) * p.Cm + row : 0;
      uint64_t mk[COLS / 64];
      if (EPI == kEpiMask) {  // before the accumulator wait: latency hidden
#pragma unroll
        for (int j = 0; j < COLS / 64; ++j) mk[j] = row_ok && j < njs ? p.mask_in[mrow + (size_t)j * p.Cm] : 0ull;
      }
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
#pragma unroll
      for (int j = 0; j < COLS / 64; ++j) {
        if (j >= njs) break;
        const int c0 = col0 + j * 64;
        const int b = sub % G::EPI_BUFS;
        uint8_t* buf = my_epi + b * 4096;
        const uint32_t rowaddr = smem_u32(buf) + lane * 128;
        uint32_t v[64];
        if (nkb > 0) {
          tmem_ld32(tbase + tcol0 + j * 64, *reinterpret_cast<uint32_t(*)[32]>(v));
          tmem_ld32(tbase + tcol0 + j * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int i = 0; i < 64; ++i) v[i] = 0u;
        }
        if (lane == 0 && sub >= G::EPI_BUFS) bulk_wait_read<G::EPI_BUFS - 1>();  // `buf`'s last store has read it
        ++sub;
        __syncwarp();
        uint64_t mword = 0;
        const uint64_t min = EPI == kEpiMask ? mk[j] : 0ull;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t qa = rowaddr + ((q ^ (lane & 7)) << 4);
          float x[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float y = __uint_as_float(v[q * 8 + i]);
            if (EPI == kEpiRelu) y = fmaxf(y, 0.f);
            if (EPI == kEpiMask) y = ((min >> (q * 8 + i)) & 1ull) ? y : 0.f;
            x[i] = y;
          }
          uint4 pk;
          __nv_bfloat162* hp = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
          for (int i = 0; i < 4; ++i) hp[i] = __floats2bfloat162_rn(x[2 * i], x[2 * i + 1]);
          if (EPI == kEpiRelu) {  // ReLU' of the stored (rounded, non-negative) value: bits != 0
            const uint32_t* w = reinterpret_cast<const uint32_t*>(&pk);
            uint32_t byte = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint32_t m = __vcmpne2(w[i], 0u);     // 0xFFFF per nonzero half
              byte |= ((m & 1u) | ((m >> 15) & 2u)) << (2 * i);
            }
            mword |= (uint64_t)byte << (q * 8);
          }
          st_shared16(qa, pk);
        }
        if (EPI == kEpiRelu && p.mask_out && row_ok) p.mask_out[mrow + (size_t)j * p.Cm] = mword;
        fence_proxy_async_smem();
        __syncwarp();
        const int x0 = n0 + c0, x1 = rbase, x2 = WGRAD ? se : p.seg0 + se;
        int sidx = 0, dseg = 0;
        if (!WGRAD && p.has_pmaps) {  // fused combine all-to-all: the owner of this segment
          const int el = x2 % p.El, c = x2 / (p.El * p.dP);
          sidx = (x2 / p.El) % p.dP;
          dseg = c * p.dE + p.dme * p.El + el;
        }
        if (!WGRAD && p.has_pmaps && sidx != p.dme) {
          // remote owner: the warp moves the box with 16-byte stores over NVLink, four
          // 128-byte row segments per instruction (rows past the segment end skipped);
          // an empty bulk group keeps the staging-buffer accounting uniform
          char* base = p.pbase[sidx] + (size_t)dseg * p.Cm * p.N * 2;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = i * 4 + (lane >> 3), q = lane & 7;
            const uint4 v = ld_shared16(smem_u32(buf) + rr * 128 + ((q ^ (rr & 7)) << 4));
            if (x1 + rr < p.Cm) *reinterpret_cast<uint4*>(base + ((size_t)(x1 + rr) * p.N + x0 + q * 8) * 2) = v;
          }
          if (lane == 0) bulk_commit();
        } else if (lane == 0) {
          if (!WGRAD && p.has_pmaps) tma_store_3d(&p.pmaps[sidx], buf, x0, x1, dseg);
          else tma_store_3d(&tmD, buf, x0, x1, x2);
          bulk_commit();
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) mbar_arrive_cluster(&tempty[acc], 0);
        else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[acc])) : "memory");
      }
      if (++acc == 2) {
        acc = 0;
        aph ^= 1;
      }
    }
    if (lane == 0) {
      bulk_wait_all();
      if (p.sig.post) asm volatile("fence.proxy.async.global;" ::: "memory");
    }
  }
  __syncwarp();
  tc_fence_before();
  if (CG == 2) cluster_sync();
  else __syncthreads();
  if (threadIdx.x == 0) sig_post_last(p.sig);  // the last CTA: every output tile is stored
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<CG>(tmem_base, TMEM_COLS);
  }
}

// ------------------------------------------------------------------ host side
static int g_reserved_sms = 0;  // SMs left to concurrent NCCL kernels (H2 in SURVEY.md)
// The calling communicator's tile counter (dynamic schedule; NULL = static): set by every
// layer entry point; the GEMMs of one communicator are stream-ordered on its caller's stream.
static thread_local unsigned int* t_tile_ctr = nullptr;
// Which GEMMs take the dynamic schedule (profiles/r02_gemm_dyn_ab.txt, per-GEMM ncu A/B at C5
// and C2).  The long-K row GEMMs (GEMM2 / dgrad2 at C5, K = 8192, 128 K-blocks per tile) gain
// 13%: under the static order the clusters drift apart (half tails end early) until the
// tiles in flight span several experts' weights and L2 thrashes (8.4 GB of DRAM reads per
// launch instead of 3.7).  GEMMs of many waves (C5's GEMM1 / dgrad1 / wgrads: >= 32 tiles per
// cluster) gain ~1% (less DRAM under the power cap); GEMMs of a few waves (C2: 3-13 tiles per
// cluster) lose 1-5% (the ticket drawn a tile ahead worsens the last wave).  LINA_GEMM_DYN=2
// forces it everywhere, 3 = the hand-off with the static order (A/B only), 0 (read at comm
// init) disables it.
static int dyn_env() {
  static const int v = [] {
    const char* e = getenv("LINA_GEMM_DYN");
    return e ? atoi(e) : 1;
  }();
  return v;
}
static bool dyn_schedule(int K, long long tiles_max, int clusters) {
  return dyn_env() >= 2 || K >= 64 * BK || tiles_max >= 32LL * clusters;
}

// SMs the persistent GEMM grid may occupy.  A persistent grid that takes every SM
// would leave the all-to-all kernels nothing to run on (they would serialise after
// it) or push a second wave of GEMM CTAs behind them.
static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    LINA_CUDA_CHECK(cudaGetDevice(&dev));
    LINA_CUDA_CHECK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  const int m = n - g_reserved_sms;
  return m < 2 ? 2 : m;
}

template <int CG, bool WGRAD, bool B_MN, int EPI, int WIDE = (EPI != kEpiNone)>
static void launch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& d, const CUtensorMap& x,
                   const TcParams& p, int grid, cudaStream_t s) {
  auto kern = tc_gemm_kernel<CG, WGRAD, B_MN, EPI, WIDE>;
  static bool attr_set = false;
  if (!attr_set) {
    LINA_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Geo<CG, WIDE>::SMEM_BYTES));
    attr_set = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(Geo<CG, WIDE>::THREADS);
  cfg.dynamicSmemBytes = Geo<CG, WIDE>::SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // (common.h: pdl_enter)
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  LINA_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, a, b, d, x, p));
}

template <int CG>
static void row_dispatch(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& md,
                         const CUtensorMap& mx, const TcParams& p, bool b_kmajor, int epi, int grid,
                         cudaStream_t s) {
  // The ReLU / mask epilogues: LINA_GEMM_WIDE=0 (4 warps, 6-stage ring), 1 (8 warps,
  // 5 stages, double-buffered boxes), 2 (8 warps, 6 stages, single-buffered boxes).
  // Default (profiles/r02_gemm_epilogue_ab.txt, ncu cycles per launch): 4 warps, except the
  // ReLU GEMM at K < 1536 (C2's K = 768: 12 K-blocks per 256 x 256 tile, the epilogue is
  // then heavy enough per flop to want 8 warps, WIDE = 2 -3.5%); at C5 (K = 2048) 4 warps
  // beat 8 by 2-6%.  (LINA_GEMM_NARROW=1 = LINA_GEMM_WIDE=0, kept for the round-2 A/B lines.)
  static const int wide_env = [] {
    const char* n = getenv("LINA_GEMM_NARROW");
    if (n && n[0] == '1') return 0;
    const char* e = getenv("LINA_GEMM_WIDE");
    if (e && (e[0] == '0' || e[0] == '1' || e[0] == '2')) return e[0] - '0';
    return -1;
  }();
  const int wide = wide_env >= 0 ? wide_env : (epi == kEpiRelu && p.K < 1536) ? 2 : 0;
  if (b_kmajor) {
    if (epi == kEpiRelu && wide == 0) launch<CG, false, false, kEpiRelu, 0>(ma, mb, md, mx, p, grid, s);
    else if (epi == kEpiRelu && wide == 1) launch<CG, false, false, kEpiRelu, 1>(ma, mb, md, mx, p, grid, s);
    else if (epi == kEpiRelu) launch<CG, false, false, kEpiRelu, 2>(ma, mb, md, mx, p, grid, s);
    else if (epi == kEpiMask) launch<CG, false, false, kEpiMask, 1>(ma, mb, md, mx, p, grid, s);
    else launch<CG, false, false, kEpiNone>(ma, mb, md, mx, p, grid, s);
  } else {
    if (epi == kEpiRelu) launch<CG, false, true, kEpiRelu, 1>(ma, mb, md, mx, p, grid, s);
    else if (epi == kEpiMask && wide == 0) launch<CG, false, true, kEpiMask, 0>(ma, mb, md, mx, p, grid, s);
    else if (epi == kEpiMask && wide == 1) launch<CG, false, true, kEpiMask, 1>(ma, mb, md, mx, p, grid, s);
    else if (epi == kEpiMask) launch<CG, false, true, kEpiMask, 2>(ma, mb, md, mx, p, grid, s);
    else launch<CG, false, true, kEpiNone>(ma, mb, md, mx, p, grid, s);
  }
}

}  // namespace tc

void tc_set_reserved_sms(int n) { tc::g_reserved_sms = n < 0 ? 0 : n; }
void tc_set_tile_counter(unsigned int* ctr) { tc::t_tile_ctr = ctr; }

// Rows per tensor-core tile (the m-block granularity launch_mtile_prefix must use).
int tc_tile_rows() { return 128 * kTcCtaGroup; }

bool tc_row_supported(const RowGemm& g) { return g.N % tc::BN == 0 && g.K % tc::BK == 0 && g.mtp; }
bool tc_wgrad_supported(const WGrad& g) { return g.M % tc_tile_rows() == 0 && g.N % tc::BN == 0; }

static void row_gemm_tc_impl(const RowGemm& g, bool b_kmajor, int epi, const PeerStore* ps,
                             cudaStream_t s);

void launch_row_gemm_tc(const RowGemm& g, bool b_kmajor, int epi, cudaStream_t s) {
  row_gemm_tc_impl(g, b_kmajor, epi, nullptr, s);
}

void launch_row_gemm_tc_peer(const RowGemm& g, bool b_kmajor, int epi, const PeerStore& ps, cudaStream_t s) {
  row_gemm_tc_impl(g, b_kmajor, epi, &ps, s);
}

std::vector<unsigned char> tc_peer_dmaps(const std::vector<char*>& bases, int N, int Cm, int nseg) {
  std::vector<unsigned char> out(bases.size() * sizeof(CUtensorMap));
  const uint64_t dims[3] = {(uint64_t)N, (uint64_t)Cm, (uint64_t)nseg};
  const uint64_t str[2] = {(uint64_t)N * 2, (uint64_t)Cm * N * 2};
  const uint32_t box[3] = {64, 32, 1};
  for (size_t r = 0; r < bases.size(); ++r) {
    CUtensorMap m = tc::make_map(bases[r], 3, dims, str, box);
    std::memcpy(out.data() + r * sizeof(CUtensorMap), &m, sizeof(CUtensorMap));
  }
  return out;
}

// tile_rows 256: 2-CTA pairs (cta_group::2, M = 256, B halves shared); 128: one CTA per
// tile (cta_group::1, M = 128) for layers whose expert segments hold few rows.
template <int CG>
static void row_gemm_tc_impl_t(const RowGemm& g, bool b_kmajor, int epi, const PeerStore* ps, cudaStream_t s);

static void row_gemm_tc_impl(const RowGemm& g, bool b_kmajor, int epi, const PeerStore* ps,
                             cudaStream_t s) {
  if (g.tile_rows == 256 && g.mtp_tail) {
    // tail split: the 256-row tiles, then the <= 128-row tails as single-CTA tiles; only the
    // second launch publishes READY (its CTAs start after the first launch has completed)
    RowGemm main = g;
    PeerSignal msig;
    if (g.sig) {
      msig = *g.sig;
      msig.post = nullptr;
      main.sig = &msig;
    }
    main.mtp_tail = nullptr;
    main.row_base = nullptr;
    row_gemm_tc_impl_t<2>(main, b_kmajor, epi, ps, s);
    RowGemm tail = g;
    tail.tile_rows = 128;
    tail.mtp = g.mtp_tail;
    tail.mtp_tail = nullptr;
    row_gemm_tc_impl_t<1>(tail, b_kmajor, epi, ps, s);
    return;
  }
  if (g.tile_rows == 128) row_gemm_tc_impl_t<1>(g, b_kmajor, epi, ps, s);
  else if (g.tile_rows == 256) row_gemm_tc_impl_t<2>(g, b_kmajor, epi, ps, s);
  else throw CudaError{"tcgen05 row GEMM: tile_rows must be 128 or 256"};
}

template <int CG>
static void row_gemm_tc_impl_t(const RowGemm& g, bool b_kmajor, int epi, const PeerStore* ps, cudaStream_t s) {
  using namespace tc;
  const int nseg_total = g.seg0 + g.nseg;  // the map spans every segment up to this launch's last
  const uint64_t adims[3] = {(uint64_t)g.K, (uint64_t)g.Cm, (uint64_t)nseg_total};
  const uint64_t astr[2] = {(uint64_t)g.K * 2, (uint64_t)g.Cm * g.K * 2};
  const uint32_t abox[3] = {BK, 128, 1};
  CUtensorMap ma = make_map(g.A, 3, adims, astr, abox);
  CUtensorMap mb;
  if (b_kmajor) {  // W [El][N][K]
    const uint64_t bd[2] = {(uint64_t)g.K, (uint64_t)(g.B_experts ? g.B_experts : g.El) * g.N};
    const uint64_t bs[1] = {(uint64_t)g.K * 2};
    const uint32_t bb[2] = {BK, (uint32_t)Geo<CG>::B_ROWS};
    mb = make_map(g.B, 2, bd, bs, bb);
  } else {  // W [El][K][N]
    const uint64_t bd[2] = {(uint64_t)g.N, (uint64_t)(g.B_experts ? g.B_experts : g.El) * g.K};
    const uint64_t bs[1] = {(uint64_t)g.N * 2};
    const uint32_t bb[2] = {64, BK};
    mb = make_map(g.B, 2, bd, bs, bb);
  }
  TcParams p{};
  p.vcount = g.vcount;
  p.mtp = g.mtp;
  p.seg_expert = g.seg_expert;
  p.seg0 = g.seg0;
  p.nseg = g.nseg;
  p.El = g.El;
  p.Cm = g.Cm;
  p.N = g.N;
  p.K = g.K;
  p.D = (__nv_bfloat16*)g.D;
  p.aux = (const __nv_bfloat16*)g.aux;
  p.mask_out = g.mask_out;
  p.mask_in = g.mask_in;
  p.row_base = g.row_base;
  if (CG == 2 && g.half_tails && !g.row_base) {  // <= 128-row last tiles as M = 128 pair tiles
    const uint32_t abox64[3] = {BK, 64, 1};
    p.tmA64 = make_map(g.A, 3, adims, astr, abox64);
    p.half = 1;
  }
  if (g.sig) p.sig = *g.sig;
  {
    const long long mt = (long long)g.nseg * ((g.Cm + Geo<CG>::ROWS - 1) / Geo<CG>::ROWS);  // m-tiles at most
    p.tile_ctr = dyn_schedule(g.K, mt * (g.N / BN), num_sms() / CG) ? t_tile_ctr : nullptr;
  }
  p.dyn_static = dyn_env() == 3;
  if (g.src_wait && !ps) {
    if (g.src_P > 32) throw CudaError{"split dispatch: at most 32 ranks"};
    p.src_wait = 1;
    p.dP = g.src_P;
    p.dme = g.src_me;
  }
  if (epi == kEpiMask && !g.mask_in) throw CudaError{"tcgen05 dgrad needs the ReLU' bit mask"};
  const uint64_t ddims[3] = {(uint64_t)g.N, (uint64_t)g.Cm, (uint64_t)nseg_total};
  const uint64_t dstr[2] = {(uint64_t)g.N * 2, (uint64_t)g.Cm * g.N * 2};
  const uint32_t dbox[3] = {64, 32, 1};
  CUtensorMap md = make_map(g.D, 3, ddims, dstr, dbox);
  CUtensorMap mx = (epi == kEpiMask) ? make_map(g.aux, 3, ddims, dstr, dbox) : md;
  if (ps) {
    if (ps->P > kMaxPeerMaps) throw CudaError{"fused transport supports at most 8 ranks"};
    std::memcpy(p.pmaps, ps->host_maps, sizeof(CUtensorMap) * ps->P);
    for (int r = 0; r < ps->P; ++r) p.pbase[r] = ps->bases[r];
    p.has_pmaps = 1;
    p.dP = ps->P;
    p.dme = ps->me;
    p.dE = ps->E;
  }
  const int grid = num_sms() / CG * CG;
  row_dispatch<CG>(ma, mb, md, mx, p, b_kmajor, epi, grid, s);
  LINA_LAUNCH_CHECK();
}

void launch_wgrad_tc(const WGrad& g, cudaStream_t s) {
  using namespace tc;
  constexpr int CG = kTcCtaGroup;
  const uint64_t nseg_total = g.nseg_total ? (uint64_t)g.nseg_total : (uint64_t)g.nchunks * g.P * g.El;
  const uint64_t ad[3] = {(uint64_t)g.M, (uint64_t)g.Cm, nseg_total};
  const uint64_t as[2] = {(uint64_t)g.M * 2, (uint64_t)g.Cm * g.M * 2};
  const uint32_t ab[3] = {64, BK, 1};
  CUtensorMap ma = make_map(g.A, 3, ad, as, ab);
  const uint64_t bd[3] = {(uint64_t)g.N, (uint64_t)g.Cm, nseg_total};
  const uint64_t bs[2] = {(uint64_t)g.N * 2, (uint64_t)g.Cm * g.N * 2};
  const uint32_t bb[3] = {64, BK, 1};
  CUtensorMap mb = make_map(g.B, 3, bd, bs, bb);
  TcParams p{};
  p.vcount = g.vcount;
  p.El = g.El;
  p.Cm = g.Cm;
  p.M = g.M;
  p.N = g.N;
  p.nchunks = g.nchunks;
  p.P = g.P;
  p.seg_range = g.seg_range;
  p.D = (__nv_bfloat16*)g.D;
  p.tile_ctr = dyn_schedule(0, (long long)g.El * (g.M / Geo<CG>::ROWS) * (g.N / BN), num_sms() / CG) ? t_tile_ctr
                                                                                                 : nullptr;
  p.dyn_static = dyn_env() == 3;
  const int tiles = g.El * (g.M / Geo<CG>::ROWS) * (g.N / BN);
  const int maxc = num_sms() / CG;
  const int grid = (tiles < maxc ? tiles : maxc) * CG;
  const uint64_t dd[3] = {(uint64_t)g.N, (uint64_t)g.M, (uint64_t)g.El};
  const uint64_t ds[2] = {(uint64_t)g.N * 2, (uint64_t)g.M * g.N * 2};
  const uint32_t db[3] = {64, 32, 1};
  CUtensorMap md = make_map(g.D, 3, dd, ds, db);
  // LINA_WGRAD_WIDE=2: 8 epilogue warps (6 stages, single-buffered boxes) — its tiles are
  // short in K (one expert's rows), so the epilogue is as heavy per flop as GEMM1's
  static const bool wide = [] {
    const char* e = getenv("LINA_WGRAD_WIDE");
    return e && e[0] == '2';
  }();
  if (wide) launch<CG, true, true, kEpiNone, 2>(ma, mb, md, md, p, grid, s);
  else launch<CG, true, true, kEpiNone>(ma, mb, md, md, p, grid, s);
  LINA_LAUNCH_CHECK();
}

}  // namespace lina
