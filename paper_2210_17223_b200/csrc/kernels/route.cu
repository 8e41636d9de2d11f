// S2 (K2): capacity slot assignment — deterministic histogram + scan + in-warp ranks.
//
// Reading R5/R6 (the paper never states capacity):
// per source rank, assignments are visited in priority order a = j*T + t (all
// first choices in token order, then all second choices, ...); slot = number of
// earlier assignments to the same expert; kept iff slot < C.
//
// Three tiny launches, all order-deterministic (atomics only count, never order):
//   count : CTA b (1024 assignments) builds a shared-memory histogram  -> blockcnt[b][E]
//   scan  : one thread per expert prefix-sums blockcnt over b            -> blockbase, counts, kept
//   assign: CTA b re-ranks its assignments with __match_any_sync (rank among
//           same-expert lanes below it) + per-warp counts prefix     -> slot[T,k], tok_of[E][C]
// tok_of[e][s] = t*k + j of the assignment holding slot s < kept[e] (entries past kept[e]
// are not written and never read): the inverse map the row-parallel permute /
// combine-backward kernels gather through.
#include <algorithm>

#include "../common.h"
#include "../kernels.h"
#include "../signal.h"

namespace lina {
namespace {

constexpr int kRouteBlock = 1024;

__global__ void __launch_bounds__(kRouteBlock) route_count_kernel(const int* __restrict__ idx, int T,
                                                                 int k, int E,
                                                                 int* __restrict__ blockcnt) {
  __shared__ int h[64];
  for (int i = threadIdx.x; i < E; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const long long a = (long long)blockIdx.x * kRouteBlock + threadIdx.x;
  if (a < (long long)T * k) {
    const int j = (int)(a / T), t = (int)(a % T);
    atomicAdd(&h[idx[(size_t)t * k + j]], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < E; i += blockDim.x) blockcnt[(size_t)blockIdx.x * E + i] = h[i];
}

__global__ void route_scan_kernel(const int* __restrict__ blockcnt, int nb, int E, int C,
                                  int* __restrict__ blockbase, int* __restrict__ counts,
                                  int* __restrict__ kept) {
  const int e = threadIdx.x;
  if (e >= E) return;
  int run = 0;
  for (int b = 0; b < nb; ++b) {
    blockbase[(size_t)b * E + e] = run;
    run += blockcnt[(size_t)b * E + e];
  }
  if (counts) counts[e] = run;
  kept[e] = run < C ? run : C;
}

__global__ void __launch_bounds__(kRouteBlock) route_assign_kernel(
    const int* __restrict__ idx, int T, int k, int E, int C, const int* __restrict__ blockbase,
    int* __restrict__ slot, int* __restrict__ tok_of) {
  __shared__ int wc[32][65];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 32 * 65; i += kRouteBlock) (&wc[0][0])[i] = 0;
  __syncthreads();
  const long long a = (long long)blockIdx.x * kRouteBlock + tid;
  const bool valid = a < (long long)T * k;
  int j = 0, t = 0, e = -1 - lane;  // distinct negative keys never match
  if (valid) {
    j = (int)(a / T);
    t = (int)(a % T);
    e = idx[(size_t)t * k + j];
  }
  const unsigned mask = __match_any_sync(0xffffffffu, e);
  const unsigned lt = (1u << lane) - 1u;
  const int rank = __popc(mask & lt);
  if (valid && lane == __ffs(mask) - 1) wc[warp][e] = __popc(mask);
  __syncthreads();
  if (valid) {
    int pre = 0;
    for (int w = 0; w < warp; ++w) pre += wc[w][e];
    const int s = blockbase[(size_t)blockIdx.x * E + e] + pre + rank;
    const int code = t * k + j;
    if (s < C) {
      slot[code] = s;
      tok_of[(size_t)e * C + s] = code;
    } else {
      slot[code] = -1;
    }
  }
}

__global__ void vcount_kernel(const int* __restrict__ recv_kept, int P, int El, int C, int n,
                              int* __restrict__ vcount, PeerSignal sig) {
  pdl_enter();
  if (threadIdx.x == 0) sig_wait(sig);  // fused transport: the peers' counts have landed
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * P * El) return;
  const int se = i % (P * El);  // s*El + el
  const int c = i / (P * El);
  const int Cm = chunk_pitch(C, n);
  const int b = chunk_begin_p(c, C, Cm), Cc = chunk_begin_p(c + 1, C, Cm) - b;
  int v = recv_kept[se] - b;
  vcount[i] = v < 0 ? 0 : (v > Cc ? Cc : v);
}

// Fused count + scan + assign (one launch): each CTA ranks its 1024 assignments within
// the block (warp match + per-warp counts), publishes its per-expert aggregate, sums the
// aggregates of all earlier CTAs (chained scan with look-back), then assigns slots.  CTAs
// take their logical index from an atomic ticket, so a CTA only waits on CTAs that have
// already started (no residency assumption).  sync = [ticket, done, flag[nb]] (zero
// between launches: the last CTA to finish resets it); agg = [nb][E] scratch.
constexpr int kRouteMaxBlocks = 4096;
__global__ void __launch_bounds__(kRouteBlock) route_fused_kernel(
    const int* __restrict__ idx, int T, int k, int E, int C, int nb, int* __restrict__ agg,
    unsigned int* __restrict__ sync, int* __restrict__ slot, int* __restrict__ tok_of, int* __restrict__ counts,
    int* __restrict__ kept, int n, int* __restrict__ vcount, int* __restrict__ mtp, int rows) {
  pdl_enter();
  __shared__ int wc[32][65];
  __shared__ int pre[64], kept_s[64];
  __shared__ unsigned int bid_s;
  unsigned int* ticket = sync;
  unsigned int* done = sync + 1;
  unsigned int* flag = sync + 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) bid_s = atomicAdd(ticket, 1u);
  for (int i = tid; i < 32 * 65; i += kRouteBlock) (&wc[0][0])[i] = 0;
  __syncthreads();
  const int b = (int)bid_s;
  const long long a = (long long)b * kRouteBlock + tid;
  const bool valid = a < (long long)T * k;
  int j = 0, t = 0, e = -1 - lane;  // distinct negative keys never match
  if (valid) {
    j = (int)(a / T);
    t = (int)(a % T);
    e = idx[(size_t)t * k + j];
  }
  const unsigned mask = __match_any_sync(0xffffffffu, e);
  const int rank = __popc(mask & ((1u << lane) - 1u));
  if (valid && lane == __ffs(mask) - 1) wc[warp][e] = __popc(mask);
  __syncthreads();
  if (tid < E) {  // this CTA's aggregate, then the exclusive prefix over earlier CTAs
    int h = 0;
    for (int w = 0; w < 32; ++w) h += wc[w][tid];
    agg[(size_t)b * E + tid] = h;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&flag[b]), "r"(1u) : "memory");
  }
  if (tid < E) pre[tid] = 0;
  __syncthreads();
  // look-back: thread i sums (earlier CTA q = i / E, expert i % E); every flag and
  // aggregate load of the CTA is in flight at once (integer adds: order-free, exact)
  for (int i = tid; i < b * E; i += kRouteBlock) {
    const int q = i / E, ee = i % E;
    unsigned int f;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(&flag[q]) : "memory");
      if (f) break;
      __nanosleep(32);
    }
    atomicAdd(&pre[ee], *((volatile const int*)&agg[(size_t)q * E + ee]));
  }
  __syncthreads();
  if (tid < E && b == nb - 1) {  // the last CTA in priority order holds the totals
    int h = 0;
    for (int w = 0; w < 32; ++w) h += wc[w][tid];
    const int tot = pre[tid] + h;
    if (counts) counts[tid] = tot;
    kept[tid] = tot < C ? tot : C;
    kept_s[tid] = tot < C ? tot : C;
  }
  // P = 1: the chunk-segment valid rows and the m-tile prefix follow from kept directly
  // (vcount / mtile_prefix kernels of the P > 1 path)
  if (vcount && b == nb - 1) {
    __syncthreads();
    const int Cm = chunk_pitch(C, n);
    for (int i = tid; i < n * E; i += kRouteBlock) {
      const int c = i / E, ee = i % E;
      const int b0 = chunk_begin_p(c, C, Cm), Cc = chunk_begin_p(c + 1, C, Cm) - b0;
      const int v = kept_s[ee] - b0;
      vcount[i] = v < 0 ? 0 : (v > Cc ? Cc : v);
    }
    __syncthreads();
    if (tid < n) {
      int run = 0;
      for (int ee = 0; ee < E; ++ee) {
        mtp[tid * (E + 1) + ee] = run;
        run += (vcount[tid * E + ee] + rows - 1) / rows;
      }
      mtp[tid * (E + 1) + E] = run;
    }
  }
  if (valid) {
    int p2 = pre[e];
    for (int w = 0; w < warp; ++w) p2 += wc[w][e];
    const int s2 = p2 + rank;
    const int code = t * k + j;
    if (s2 < C) {
      slot[code] = s2;
      tok_of[(size_t)e * C + s2] = code;
    } else {
      slot[code] = -1;
    }
  }
  __syncthreads();
  if (tid == 0) {  // the last CTA to finish re-arms the sync words for the next launch
    __threadfence();
    if (atomicAdd(done, 1u) == (unsigned)nb - 1u) {
      for (int q = 0; q < nb; ++q) flag[q] = 0u;
      *ticket = 0u;
      __threadfence();
      *done = 0u;
    }
  }
}

// One thread waits for the peers' flags; the consumer kernel follows in stream order.
// Waiting in a 1-CTA kernel (not in every CTA of the consumer) keeps the SMs free for
// kernels the peers' progress may depend on (e.g. an NCCL allreduce on another stream).
__global__ void sig_wait_kernel(PeerSignal sig) {
  pdl_wait();  // (its successor is released only after the flags: no CTAs parked beside a spin)
  if (threadIdx.x == 0) {
    sig_wait(sig);
    sig_post(sig);                      // (a 1-CTA kernel publishes right away)
    if (sig.bump) *sig.bump = *sig.bump + 1u;
  }
}

__global__ void mtile_prefix_kernel(const int* __restrict__ vcount, int n, int nseg, int rows,
                                    int* __restrict__ mtp) {
  pdl_enter();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  int run = 0;
  for (int i = 0; i < nseg; ++i) {
    mtp[c * (nseg + 1) + i] = run;
    run += (vcount[c * nseg + i] + rows - 1) / rows;
  }
  mtp[c * (nseg + 1) + nseg] = run;
}

__global__ void mtile_split_kernel(const int* __restrict__ vcount, int n, int nseg, int* __restrict__ mtp,
                                   int* __restrict__ mtpt, int* __restrict__ rbase) {
  pdl_enter();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  int run = 0, runt = 0;
  for (int i = 0; i < nseg; ++i) {
    const int v = vcount[c * nseg + i], full = v / 256, rem = v % 256;
    mtp[c * (nseg + 1) + i] = run;
    mtpt[c * (nseg + 1) + i] = runt;
    rbase[c * nseg + i] = full * 256;
    run += full + (rem > 128 ? 1 : 0);
    runt += (rem > 0 && rem <= 128) ? 1 : 0;
  }
  mtp[c * (nseg + 1) + nseg] = run;
  mtpt[c * (nseg + 1) + nseg] = runt;
}

}  // namespace

void launch_mtile_split(const int* vcount, int n, int nseg, int* mtp, int* mtp_tail, int* rbase, cudaStream_t s) {
  if (n <= 0) return;
  launch_k(mtile_split_kernel, dim3((n + 63) / 64), dim3(64), 0, s, vcount, n, nseg, mtp, mtp_tail, rbase);
  LINA_LAUNCH_CHECK();
}

void launch_mtile_prefix(const int* vcount, int n, int nseg, int rows, int* mtp, cudaStream_t s) {
  if (n <= 0) return;
  launch_k(mtile_prefix_kernel, dim3((n + 63) / 64), dim3(64), 0, s, vcount, n, nseg, rows, mtp);
  LINA_LAUNCH_CHECK();
}

void launch_sig_wait(const PeerSignal& sig, cudaStream_t s) {
  if (!sig.wait && !sig.post && !sig.bump) return;
  launch_k(sig_wait_kernel, dim3(1), dim3(32), 0, s, sig);
  LINA_LAUNCH_CHECK();
}

void launch_vcount(const int* recv_kept, int P, int El, int C, int n, int* vcount, cudaStream_t s,
                   const PeerSignal* sig) {
  const int tot = n * P * El;
  if (tot <= 0 && !sig) return;
  launch_k(vcount_kernel, dim3(std::max(1, (tot + 255) / 256)), dim3(256), 0, s, recv_kept, P, El, C, n, vcount,
           sig ? *sig : PeerSignal{});
  LINA_LAUNCH_CHECK();
}

size_t route_sync_words() { return 2 + kRouteMaxBlocks; }

size_t route_scratch_ints(int T, int k, int E) {
  const long long nb = ((long long)T * k + kRouteBlock - 1) / kRouteBlock;
  return (size_t)(2 * nb * E);
}

void launch_route(const int* idx, int T, int k, int E, int C, int* scratch, int* slot, int* counts,
                  int* kept, int* tok_of, cudaStream_t s, unsigned int* sync, int n_chunks, int* vcount, int* mtp,
                  int tile_rows) {
  // tok_of[e][s] is written for every kept slot s < kept[e]; readers never look past kept[e]
  if (T <= 0) {
    LINA_CUDA_CHECK(cudaMemsetAsync(kept, 0, sizeof(int) * E, s));
    if (counts) LINA_CUDA_CHECK(cudaMemsetAsync(counts, 0, sizeof(int) * E, s));
    if (vcount) {
      launch_vcount(kept, 1, E, C, n_chunks, vcount, s);
      launch_mtile_prefix(vcount, n_chunks, E, tile_rows, mtp, s);
    }
    return;
  }
  const int nb = (int)(((long long)T * k + kRouteBlock - 1) / kRouteBlock);
  if (sync && nb <= kRouteMaxBlocks) {
    launch_k(route_fused_kernel, dim3(nb), dim3(kRouteBlock), 0, s, idx, T, k, E, C, nb, scratch, sync, slot, tok_of,
             counts, kept, n_chunks, vcount, mtp, tile_rows);
    LINA_LAUNCH_CHECK();
    return;
  }
  int* blockcnt = scratch;
  int* blockbase = scratch + (size_t)nb * E;
  route_count_kernel<<<nb, kRouteBlock, 0, s>>>(idx, T, k, E, blockcnt);
  LINA_LAUNCH_CHECK();
  route_scan_kernel<<<1, 64, 0, s>>>(blockcnt, nb, E, C, blockbase, counts, kept);
  LINA_LAUNCH_CHECK();
  route_assign_kernel<<<nb, kRouteBlock, 0, s>>>(idx, T, k, E, C, blockbase, slot, tok_of);
  LINA_LAUNCH_CHECK();
  if (vcount) {
    launch_vcount(kept, 1, E, C, n_chunks, vcount, s);
    launch_mtile_prefix(vcount, n_chunks, E, tile_rows, mtp, s);
  }
}

}  // namespace lina
