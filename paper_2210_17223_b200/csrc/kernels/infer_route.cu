// S10: replica routing for inference (§5.2, §6.2).
//
// After the plan is fixed (identical on every rank), source rank s sends the
// c_{s,e} tokens it routed to expert e, in slot order, as r_e contiguous blocks whose
// sizes differ by at most one; block q goes to replica (q + s) mod r_e, i.e. device
// replica_device[e][(q + s) mod r_e] ("how many tokens each replica should handle to
// balance the load"; reading R14).  The send buffer is ordered by destination
// device, then by the experts that device hosts (ascending), so every (device,
// expert) block is one contiguous ncclSend of the unequal-split all-to-all.
//
// infer_permute: one warp per (token, choice): row = send_off[dv][e] + offset in its
//                block; copies the token row (16-byte vectors) and records the row for
//                the combine.
// combine_rows : y_t = Σ_j g_tj · Back[arow[t,j]] (fp32 accumulate, j ascending, R9).
// regroup      : the rows a device receives arrive source-major (one message per peer:
//                [src][hosted expert][rows]); the expert GEMMs want them expert-major
//                ([hosted expert][Cm] with every source's rows contiguous), so each
//                expert is one segment padded once to the tile height instead of once
//                per source.  The same kernel moves the outputs back.
#include <algorithm>

#include "../common.h"
#include "../kernels.h"
#include "../signal.h"

namespace lina {
namespace {

// tables (int32): r[E] | rdev[E][N] | send_off[N][E] | cnt[E] (this source's counts)
template <typename T>
__global__ void infer_permute_kernel(const T* __restrict__ X, const int* __restrict__ idx,
                                     const int* __restrict__ slot, const int* __restrict__ tab,
                                     int Tn, int k, int d, int E, int N, int s, T* __restrict__ Send,
                                     int* __restrict__ arow) {
  const long long a = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (a >= (long long)Tn * k) return;
  const int* r_e = tab;
  const int* rdev = tab + E;
  const int* send_off = rdev + (size_t)E * N;
  const int* cnt = send_off + (size_t)N * E;
  const int e = idx[a], sl = slot[a];
  const int r = r_e[e], c = cnt[e];
  const int base = c / r, extra = c % r;
  // block q of slot sl: the first `extra` blocks hold base+1 slots
  int q, start;
  if (sl < extra * (base + 1)) {
    q = sl / (base + 1);
    start = q * (base + 1);
  } else {
    q = extra + (sl - extra * (base + 1)) / base;
    start = extra * (base + 1) + (q - extra) * base;
  }
  const int dv = rdev[(size_t)e * N + (q + s) % r];
  const int row = send_off[(size_t)dv * E + e] + (sl - start);
  if (lane == 0) arow[a] = row;
  constexpr int V = 16 / sizeof(T);
  const uint4* src = reinterpret_cast<const uint4*>(X + (size_t)(a / k) * d);
  uint4* dst = reinterpret_cast<uint4*>(Send + (size_t)row * d);
  for (int v = lane; v < d / V; v += 32) dst[v] = src[v];
}

template <typename T>
__global__ void combine_rows_kernel(const T* __restrict__ Back, const int* __restrict__ arow,
                                    const float* __restrict__ gate, int Tn, int k, int d,
                                    T* __restrict__ Y) {
  const long long t = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= Tn) return;
  constexpr int V = 16 / sizeof(T);
  const T* rowp[8];
  float g[8];
  for (int j = 0; j < k; ++j) {
    rowp[j] = Back + (size_t)arow[t * k + j] * d;
    g[j] = gate[t * k + j];
  }
#pragma unroll 4
  for (int v = lane; v < d / V; v += 32) {
    float acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0.f;
    for (int j = 0; j < k; ++j) {
      float x[V];
      load16(rowp[j] + v * V, x, (const T*)nullptr);
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] = fmaf(g[j], x[i], acc[i]);
    }
    store16(Y + t * d + v * V, acc, (T*)nullptr);
  }
}

inline int blocks_for_warps(long long warps) { return (int)((warps * 32 + 255) / 256); }


// rows of segment (src, hh): source-major at off_sm(src, hh) (row-major prefix over
// [P][mpd]); expert-major at hh*Cm + Σ_{s' < src} nrecv[s'][hh].
template <typename T>
__global__ void __launch_bounds__(256) regroup_kernel(const T* __restrict__ src_buf, T* __restrict__ dst_buf,
                                                      const int* __restrict__ nrecv, int P, int mpd, int Cm,
                                                      int d, int to_expert_major) {
  __shared__ long long off_sm, off_em;
  __shared__ int nrows;
  const int seg = blockIdx.y, sidx = seg / mpd, hh = seg % mpd;
  if (threadIdx.x == 0) {
    long long a = 0, b = 0;
    for (int i = 0; i < seg; ++i) a += nrecv[i];
    for (int s2 = 0; s2 < sidx; ++s2) b += nrecv[s2 * mpd + hh];
    off_sm = a;
    off_em = (long long)hh * Cm + b;
    nrows = nrecv[seg];
  }
  __syncthreads();
  constexpr int V = 16 / sizeof(T);
  const int nv = d / V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = blockIdx.x * 8 + warp; i < nrows; i += gridDim.x * 8) {
    const long long rs = off_sm + i, re = off_em + i;
    const uint4* from = reinterpret_cast<const uint4*>(src_buf + (size_t)(to_expert_major ? rs : re) * d);
    uint4* to = reinterpret_cast<uint4*>(dst_buf + (size_t)(to_expert_major ? re : rs) * d);
    for (int v = lane; v < nv; v += 32) to[v] = from[v];
  }
}

// blocks[b] = {src_row, dst_row, nrows}: rows of block b go to peer_dst[b] (blockIdx.y = b)
template <typename T>
__global__ void __launch_bounds__(256) push_blocks_kernel(const T* __restrict__ src, T* const* __restrict__ peer_dst,
                                                          const int* __restrict__ blocks, int d, PeerSignal sig) {
  pdl_enter();
  const int b = blockIdx.y;
  const int r0 = blocks[3 * b], d0 = blocks[3 * b + 1], n = blocks[3 * b + 2];
  constexpr int V = 16 / sizeof(T);
  const int nv = d / V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* dst = peer_dst[b];
  for (int i = blockIdx.x * 8 + warp; i < n; i += gridDim.x * 8) {
    const uint4* from = reinterpret_cast<const uint4*>(src + (size_t)(r0 + i) * d);
    uint4* to = reinterpret_cast<uint4*>(dst + (size_t)(d0 + i) * d);
    for (int v = lane; v < nv; v += 32) to[v] = from[v];
  }
  __syncthreads();
  if (threadIdx.x == 0) sig_post_last(sig);
}
}  // namespace

void launch_infer_permute(int dtype, const void* X, const int* idx, const int* slot, const int* tab,
                          int T, int k, int d, int E, int N, int s, void* Send, int* arow,
                          cudaStream_t st) {
  const long long n = (long long)T * k;
  if (n <= 0) return;
  if (dtype == 0)
    infer_permute_kernel<float><<<blocks_for_warps(n), 256, 0, st>>>(
        (const float*)X, idx, slot, tab, T, k, d, E, N, s, (float*)Send, arow);
  else
    infer_permute_kernel<__nv_bfloat16><<<blocks_for_warps(n), 256, 0, st>>>(
        (const __nv_bfloat16*)X, idx, slot, tab, T, k, d, E, N, s, (__nv_bfloat16*)Send, arow);
  LINA_LAUNCH_CHECK();
}

void launch_combine_rows(int dtype, const void* Back, const int* arow, const float* gate, int T, int k,
                         int d, void* Y, cudaStream_t st) {
  if (T <= 0) return;
  if (dtype == 0)
    combine_rows_kernel<float><<<blocks_for_warps(T), 256, 0, st>>>((const float*)Back, arow, gate, T,
                                                                     k, d, (float*)Y);
  else
    combine_rows_kernel<__nv_bfloat16><<<blocks_for_warps(T), 256, 0, st>>>(
        (const __nv_bfloat16*)Back, arow, gate, T, k, d, (__nv_bfloat16*)Y);
  LINA_LAUNCH_CHECK();
}

}  // namespace lina

namespace lina {
void launch_regroup(int dtype, const void* src, void* dst, const int* nrecv, int P, int mpd, int Cm, int d,
                    int max_rows, bool to_expert_major, cudaStream_t st) {
  if (max_rows <= 0 || P * mpd == 0) return;
  dim3 grid(std::min(64, (max_rows + 7) / 8), P * mpd);
  if (dtype == 0)
    regroup_kernel<float><<<grid, 256, 0, st>>>((const float*)src, (float*)dst, nrecv, P, mpd, Cm, d,
                                               to_expert_major ? 1 : 0);
  else
    regroup_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)src, (__nv_bfloat16*)dst, nrecv,
                                                         P, mpd, Cm, d, to_expert_major ? 1 : 0);
  LINA_LAUNCH_CHECK();
}
}  // namespace lina

namespace lina {
void launch_push_blocks(int dtype, const void* src, void* const* peer_dst, const int* blocks, int P, int d,
                        int max_rows, const PeerSignal& sig, cudaStream_t st) {
  dim3 grid(std::max(1, std::min(64, (max_rows + 7) / 8)), P);
  if (dtype == 0)
    launch_k(push_blocks_kernel<float>, grid, dim3(256), 0, st, (const float*)src, (float* const*)peer_dst, blocks, d,
             sig);
  else
    launch_k(push_blocks_kernel<__nv_bfloat16>, grid, dim3(256), 0, st, (const __nv_bfloat16*)src,
             (__nv_bfloat16* const*)peer_dst, blocks, d, sig);
  LINA_LAUNCH_CHECK();
}
}  // namespace lina
