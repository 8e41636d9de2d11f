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
// (dL, dX and dWg are in gate_bwd.cu.)
// Rows are moved as 16-byte vectors, one warp per row / token.
#include <algorithm>

#include "../common.h"
#include "../kernels.h"
#include "../signal.h"

namespace lina {
namespace {

// Warps move R whole rows at a time: the row indices are resolved by the first R lanes
// and broadcast, then all R x NVL 16-byte loads of a lane are issued before the first
// store (NVL = vectors per lane per row, <= kLoadsPerLane loads in flight per lane).
// NVL = 0 instantiates the plain strided loop for rows wider than 8 x 32 vectors.
constexpr int kLoadsPerLane = 12;

__device__ __forceinline__ size_t peer_row(int c, int e, int r, int El, int P, int me, int Cm) {
  return (((size_t)c * P + me) * El + (e % El)) * Cm + r;
}

// Send-layout row gw = (c*E + e)*Cm + r -> the assignment code in it (-1 = padding) and,
// for the fused dispatch, its destination (owner e / El, receive row peer_row(...)).
// kRowSkip: a padding row past the first 64-row block boundary after the segment's valid
// rows.  Only rows [v, roundup64(v)) of a segment are ever read as padding (the wgrad
// K-blocks are 64 rows; rows past them only feed output rows nobody reads), so only
// those are written as zeros — padding is ~20% of the rows at cf = 1.25, and at P > 1
// it would cross NVLink.
constexpr int kRowSkip = -2;
__device__ __forceinline__ int row_assignment(long long gw, const int* __restrict__ tok_of,
                                              const int* __restrict__ kept, int E, int C, int Cm, int El, int P,
                                              int me, int& owner, size_t& prow) {
  const int r = (int)(gw % Cm);
  const int ce = (int)(gw / Cm);
  const int e = ce % E, c = ce / E;
  const int b = chunk_begin_p(c, C, Cm), Cc = chunk_begin_p(c + 1, C, Cm) - b;
  owner = El > 0 ? e / El : 0;
  prow = El > 0 ? peer_row(c, e, r, El, P, me, Cm) : (size_t)gw;
  const int v = min(max(kept[e] - b, 0), Cc);  // valid rows of this (chunk, expert) segment
  const int a = (r < v) ? tok_of[(size_t)e * C + b + r] : -1;  // slots >= kept[e] are never read
  if (a < 0) {
    if (r >= min(Cm, (v + 63) & ~63)) return kRowSkip;  // (the segment pitch Cm, not Cc, bounds the read)
  }
  return a;
}

// First row of this warp's R-row group (-1: none).  Peer stores: warps are rotated so
// that every rank starts with the rows of owner (me + 1) % P — at any moment the P ranks
// write to P different owners instead of all to owner 0 (no incast on one rank's links).
template <bool PEER>
__device__ __forceinline__ long long rotated_row0(int R, long long rows, int El, int P, int me, int Cm) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = (rows + R - 1) / R;
  if (w >= nw) return -1;
  long long wr = w;
  if (PEER && P > 1) {
    wr += ((long long)((me + 1) % P) * El * Cm) / R;
    if (wr >= nw) wr -= nw;
  }
  return wr * R;
}

// permute (PEER = false): Send[row] = X[token of row] or 0.
// fused dispatch (PEER = true): the same rows stored straight into the owners' receive
// buffers over NVLink (peer[o] = rank o's buffer mapped here): row (c, e, r) lands at
// recv row ((c*P + me)*El + e%El)*Cm + r of owner o = e / El, so the permute IS the
// dispatch all-to-all.
template <int NVL>
constexpr int permute_R() { return NVL == 0 ? 1 : (NVL >= kLoadsPerLane ? 1 : kLoadsPerLane / NVL); }

// The R rows [g0 + row0, g0 + min(row0 + R, rows)) of one warp.
template <typename T, int NVL, bool PEER>
__device__ __forceinline__ void permute_rows_at(const T* __restrict__ X, const int* __restrict__ tok_of,
                                                const int* __restrict__ kept, int k, int d, int E, int C,
                                                long long g0, long long row0, long long rows, int Cm, int El,
                                                int P, int me, T* __restrict__ Send, T* const* __restrict__ peer) {
  constexpr int R = permute_R<NVL>();
  constexpr int NL = NVL == 0 ? 1 : NVL;
  constexpr int V = 16 / sizeof(T);
  const int lane = threadIdx.x & 31;
  const int nv = d / V;
  int a = -1, owner = 0;
  size_t prow = 0;
  if (lane < R && row0 + lane < rows)
    a = row_assignment(g0 + row0 + lane, tok_of, kept, E, C, Cm, PEER ? El : 0, P, me, owner, prow);
  if constexpr (NVL == 0) {
    uint4* dst = reinterpret_cast<uint4*>(PEER ? peer[owner] + prow * d : Send + (size_t)(g0 + row0) * d);
    a = __shfl_sync(0xffffffffu, a, 0);
    if (a == kRowSkip) return;
    dst = reinterpret_cast<uint4*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(dst), 0));
    const uint4* src = reinterpret_cast<const uint4*>(X + (size_t)(a >= 0 ? a / k : 0) * d);
    for (int v = lane; v < nv; v += 32) dst[v] = a >= 0 ? src[v] : make_uint4(0, 0, 0, 0);
  } else {
    uint4 buf[R][NL];
    int ai[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      ai[i] = __shfl_sync(0xffffffffu, a, i);
      const uint4* src = reinterpret_cast<const uint4*>(X + (size_t)(ai[i] >= 0 ? ai[i] / k : 0) * d);
#pragma unroll
      for (int j = 0; j < NL; ++j) {
        const int v = lane + 32 * j;
        buf[i][j] = (ai[i] >= 0 && v < nv) ? src[v] : make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      if (row0 + i >= rows) break;
      if (ai[i] == kRowSkip) continue;
      uint4* dst;
      if constexpr (PEER) {
        const int o = __shfl_sync(0xffffffffu, owner, i);
        const size_t pr = __shfl_sync(0xffffffffu, (unsigned long long)prow, i);
        dst = reinterpret_cast<uint4*>(peer[o] + pr * d);
      } else {
        dst = reinterpret_cast<uint4*>(Send + (size_t)(g0 + row0 + i) * d);
      }
#pragma unroll
      for (int j = 0; j < NL; ++j) {
        const int v = lane + 32 * j;
        if (v < nv) dst[v] = buf[i][j];
      }
    }
  }
}

template <typename T, int NVL, bool PEER>
__device__ __forceinline__ void permute_rows(const T* __restrict__ X, const int* __restrict__ tok_of,
                                             const int* __restrict__ kept, int k, int d, int E, int C, int c0,
                                             int nc, int Cm, int El, int P, int me, T* __restrict__ Send,
                                             T* const* __restrict__ peer) {
  const long long rows = (long long)nc * E * Cm;  // the micro-op chunks [c0, c0 + nc)
  const long long g0 = (long long)c0 * E * Cm;
  const long long row0 = rotated_row0<PEER>(permute_R<NVL>(), rows, El, P, me, Cm);
  if (row0 < 0) return;
  permute_rows_at<T, NVL, PEER>(X, tok_of, kept, k, d, E, C, g0, row0, rows, Cm, El, P, me, Send, peer);
}

template <typename T, int NVL, bool PEER>
__global__ void __launch_bounds__(256) permute_kernel(const T* __restrict__ X, const int* __restrict__ tok_of,
                                                      int k, int d, int E, int C, int c0, int nc, int Cm,
                                                      int El, int P, int me, T* __restrict__ Send,
                                                      T* const* __restrict__ peer, const int* __restrict__ kept,
                                                      int* const* __restrict__ peer_counts, PeerSignal sig) {
  pdl_enter();
  if constexpr (PEER) {
    // the owners' receive buffers are free (their FREE of this round), then this rank's
    // counts go to every owner's recv_kept
    if (threadIdx.x == 0) sig_wait(sig);
    __syncthreads();
    if (blockIdx.x == 0 && c0 == 0)
      for (int i = threadIdx.x; i < P * El; i += blockDim.x) peer_counts[i / El][me * El + i % El] = kept[i];
  }
  permute_rows<T, NVL, PEER>(X, tok_of, kept, k, d, E, C, c0, nc, Cm, El, P, me, Send, peer);
  if constexpr (PEER) {
    __syncthreads();
    if (threadIdx.x == 0) sig_post_last(sig);  // the last CTA: READY of the dispatch
  }
}

template <typename T, int NVL, int KT>
__device__ __forceinline__ void combine_tokens(const T* __restrict__ Recv, const int* __restrict__ idx,
                                               const int* __restrict__ slot, const float* __restrict__ gate,
                                               int Tn, int k, int d, int E, int C, int n, int Cm,
                                               T* __restrict__ Y, const int* __restrict__ ebase) {
  constexpr int NL = NVL > 0 ? NVL : 1;  // (NVL = 0 is never launched)
  constexpr int U = kLoadsPerLane / NL;
  constexpr int TP = U / KT > 0 ? U / KT : 1;
  static_assert(TP * KT <= 32, "pairs per warp");
  constexpr int V = 16 / sizeof(T);
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long t0 = w * TP;
  if (t0 >= Tn) return;
  const int nv = d / V;
  // lane q <-> pair (t0 + q / KT, q % KT)
  size_t rowq = 0;
  float gq = 0.f;
  bool kq = false;
  if (lane < TP * KT && t0 + lane / KT < Tn) {
    const size_t pi = (size_t)t0 * KT + lane;
    const int s = slot[pi];
    kq = s >= 0;
    if (kq) {
      rowq = ebase ? (size_t)(ebase[idx[pi]] + s) : send_row(idx[pi], s, E, C, n, Cm);  // (dropless: compact)
      gq = gate[pi];
    }
  }
  uint4 buf[TP * KT][NL];
  bool kept[TP * KT];
  float g[TP * KT];
#pragma unroll
  for (int q = 0; q < TP * KT; ++q) {
    kept[q] = __shfl_sync(0xffffffffu, (int)kq, q);
    g[q] = __shfl_sync(0xffffffffu, gq, q);
    const size_t rq = __shfl_sync(0xffffffffu, (unsigned long long)rowq, q);
    const uint4* src = reinterpret_cast<const uint4*>(Recv + rq * d);
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      const int v = lane + 32 * j;
      buf[q][j] = (kept[q] && v < nv) ? src[v] : make_uint4(0, 0, 0, 0);
    }
  }
#pragma unroll
  for (int i = 0; i < TP; ++i) {
    if (t0 + i >= Tn) break;
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      const int v = lane + 32 * j;
      if (v >= nv) continue;
      float acc[V];
#pragma unroll
      for (int u = 0; u < V; ++u) acc[u] = 0.f;
#pragma unroll
      for (int q = i * KT; q < (i + 1) * KT; ++q) {
        if (!kept[q]) continue;
        float x[V];
        load16(&buf[q][j], x, (const T*)nullptr);
#pragma unroll
        for (int u = 0; u < V; ++u) acc[u] = fmaf(g[q], x[u], acc[u]);
      }
      store16(Y + (size_t)(t0 + i) * d + v * V, acc, (T*)nullptr);
    }
  }
}

// combine: y_t = Σ_{j kept, ascending} g_tj · Recv[row(t, j)] (fp32 accumulation).  A warp
// owns TP = U / k tokens (U = kLoadsPerLane / NVL rows in flight); lane q < TP*k resolves
// pair q, then every row load is issued before the sums.
template <typename T, int NVL, int KT>
__global__ void __launch_bounds__(256) combine_kernel(const T* __restrict__ Recv, const int* __restrict__ idx,
                                                      const int* __restrict__ slot,
                                                      const float* __restrict__ gate, int Tn, int k, int d,
                                                      int E, int C, int n, int Cm, T* __restrict__ Y,
                                                      PeerSignal sig, const int* __restrict__ ebase) {
  pdl_enter();
  // fused transport: this rank's backward receive buffers are free again (block 0 posts);
  // the peers' returned expert outputs have landed (every CTA waits)
  if (blockIdx.x == 0 && threadIdx.x == 0) sig_post(sig);
  if (sig.wait) {
    if (threadIdx.x == 0) sig_wait(sig);
    __syncthreads();
  }
  combine_tokens<T, NVL, KT>(Recv, idx, slot, gate, Tn, k, d, E, C, n, Cm, Y, ebase);
  if (sig.bump) {  // the forward's last kernel closes its round
    __syncthreads();
    if (threadIdx.x == 0) sig_bump_last(sig);
  }
}

template <typename T>
__device__ __forceinline__ void combine_token_loop(const T* __restrict__ Recv, const int* __restrict__ idx,
                                                   const int* __restrict__ slot, const float* __restrict__ gate,
                                                   long long t, int lane, int k, int d, int E, int C, int n,
                                                   int Cm, T* __restrict__ Y, const int* __restrict__ ebase) {
  constexpr int V = 16 / sizeof(T);
  const T* rowp[8];
  float g[8];
  int kk = 0;
  for (int j = 0; j < k; ++j) {
    const int s = slot[t * k + j];
    if (s >= 0) {
      rowp[kk] = Recv + (ebase ? (size_t)(ebase[idx[t * k + j]] + s) : send_row(idx[t * k + j], s, E, C, n, Cm)) * d;
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

// generic k / wide rows: one warp per token, strided loop
template <typename T>
__global__ void combine_loop_kernel(const T* __restrict__ Recv, const int* __restrict__ idx,
                                    const int* __restrict__ slot, const float* __restrict__ gate,
                                    int Tn, int k, int d, int E, int C, int n, int Cm,
                                    T* __restrict__ Y, PeerSignal sig, const int* __restrict__ ebase) {
  pdl_enter();
  if (blockIdx.x == 0 && threadIdx.x == 0) sig_post(sig);
  if (sig.wait) {
    if (threadIdx.x == 0) sig_wait(sig);
    __syncthreads();
  }
  const long long t = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t < Tn) combine_token_loop<T>(Recv, idx, slot, gate, t, lane, k, d, E, C, n, Cm, Y, ebase);
  if (sig.bump) {
    __syncthreads();
    if (threadIdx.x == 0) sig_bump_last(sig);
  }
}

// combine backward over send-layout rows: dg_a = <dY_t, O_row>, dSend[row] = g_a · dY_t
// (0 for padding rows).  PEER: dSend rows are stored into the owners' receive buffers.
template <int NVL>
constexpr int combine_bwd_R() { return NVL == 0 ? 1 : (2 * NVL >= kLoadsPerLane ? 1 : kLoadsPerLane / (2 * NVL)); }

template <typename T, int NVL, bool PEER>
__device__ __forceinline__ void combine_bwd_rows_at(const T* __restrict__ dY, const T* __restrict__ Recv,
                                                    const int* __restrict__ tok_of, const int* __restrict__ kept,
                                                    const float* __restrict__ gate, int k, int d, int E, int C,
                                                    long long g0, long long row0, long long rows, int Cm, int El,
                                                    int P, int me, T* __restrict__ dSend,
                                                    T* const* __restrict__ peer, float* __restrict__ dg) {
  constexpr int NL = NVL == 0 ? 1 : NVL;
  constexpr int R = combine_bwd_R<NVL>();
  constexpr int V = 16 / sizeof(T);
  const int lane = threadIdx.x & 31;
  const int nv = d / V;
  int a = -1, owner = 0;
  size_t prow = 0;
  float ga = 0.f;
  if (lane < R && row0 + lane < rows) {
    a = row_assignment(g0 + row0 + lane, tok_of, kept, E, C, Cm, PEER ? El : 0, P, me, owner, prow);
    if (a >= 0) ga = gate[a];
  }
  if constexpr (NVL == 0) {
    a = __shfl_sync(0xffffffffu, a, 0);
    if (a == kRowSkip) return;
    ga = __shfl_sync(0xffffffffu, ga, 0);
    owner = __shfl_sync(0xffffffffu, owner, 0);
    prow = __shfl_sync(0xffffffffu, (unsigned long long)prow, 0);
    T* dst = PEER ? peer[owner] + prow * d : dSend + (size_t)(g0 + row0) * d;
    if (a < 0) {
      for (int v = lane; v < nv; v += 32) reinterpret_cast<uint4*>(dst)[v] = make_uint4(0, 0, 0, 0);
      return;
    }
    const T* dy = dY + (size_t)(a / k) * d;
    const T* o = Recv + (size_t)(g0 + row0) * d;
    float dot = 0.f;
    for (int v = lane; v < nv; v += 32) {
      float x[V], y[V];
      load16(dy + v * V, x, (const T*)nullptr);
      load16(o + v * V, y, (const T*)nullptr);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        dot = fmaf(x[i], y[i], dot);
        x[i] *= ga;
      }
      store16(dst + v * V, x, (T*)nullptr);
    }
#pragma unroll
    for (int o2 = 16; o2; o2 >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o2);
    if (lane == 0) dg[a] = dot;
  } else {
    uint4 by[R][NL], bo[R][NL];
    int ai[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      ai[i] = __shfl_sync(0xffffffffu, a, i);
      const uint4* dy = reinterpret_cast<const uint4*>(dY + (size_t)(ai[i] >= 0 ? ai[i] / k : 0) * d);
      const uint4* o = reinterpret_cast<const uint4*>(Recv + (size_t)(g0 + (row0 + i < rows ? row0 + i : 0)) * d);
#pragma unroll
      for (int j = 0; j < NL; ++j) {
        const int v = lane + 32 * j;
        const bool ok = ai[i] >= 0 && v < nv;
        by[i][j] = ok ? dy[v] : make_uint4(0, 0, 0, 0);
        bo[i][j] = ok ? o[v] : make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      if (row0 + i >= rows) break;
      if (ai[i] == kRowSkip) continue;
      const float g = __shfl_sync(0xffffffffu, ga, i);
      T* dst;
      if constexpr (PEER) {
        const int o = __shfl_sync(0xffffffffu, owner, i);
        const size_t pr = __shfl_sync(0xffffffffu, (unsigned long long)prow, i);
        dst = peer[o] + pr * d;
      } else {
        dst = dSend + (size_t)(g0 + row0 + i) * d;
      }
      float dot = 0.f;
#pragma unroll
      for (int j = 0; j < NL; ++j) {
        const int v = lane + 32 * j;
        if (v >= nv) continue;
        float x[V], y[V];
        load16(&by[i][j], x, (const T*)nullptr);
        load16(&bo[i][j], y, (const T*)nullptr);
#pragma unroll
        for (int u = 0; u < V; ++u) {
          dot = fmaf(x[u], y[u], dot);
          x[u] *= g;
        }
        store16(dst + v * V, x, (T*)nullptr);
      }
#pragma unroll
      for (int o2 = 16; o2; o2 >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o2);
      if (lane == 0 && ai[i] >= 0) dg[ai[i]] = dot;
    }
  }
}

template <typename T, int NVL, bool PEER>
__device__ __forceinline__ void combine_bwd_rows(const T* __restrict__ dY, const T* __restrict__ Recv,
                                                 const int* __restrict__ tok_of, const int* __restrict__ kept,
                                                 const float* __restrict__ gate,
                                                 int k, int d, int E, int C, int c0, int nc, int Cm, int El, int P,
                                                 int me,
                                                 T* __restrict__ dSend, T* const* __restrict__ peer,
                                                 float* __restrict__ dg) {
  const long long rows = (long long)nc * E * Cm;  // the micro-op chunks [c0, c0 + nc)
  const long long g0 = (long long)c0 * E * Cm;
  const long long row0 = rotated_row0<PEER>(combine_bwd_R<NVL>(), rows, El, P, me, Cm);
  if (row0 < 0) return;
  combine_bwd_rows_at<T, NVL, PEER>(dY, Recv, tok_of, kept, gate, k, d, E, C, g0, row0, rows, Cm, El, P, me, dSend,
                                    peer, dg);
}

template <typename T, int NVL, bool PEER>
__global__ void __launch_bounds__(256) combine_bwd_kernel(const T* __restrict__ dY, const T* __restrict__ Recv,
                                                          const int* __restrict__ tok_of,
                                                          const int* __restrict__ kept,
                                                          const float* __restrict__ gate, int k, int d,
                                                          int E, int C, int c0, int nc, int Cm, int El, int P,
                                                          int me, T* __restrict__ dSend,
                                                          T* const* __restrict__ peer,
                                                          float* __restrict__ dg, PeerSignal sig) {
  pdl_enter();
  if constexpr (PEER) {  // the owners' backward receive buffers are free (their FREE)
    if (threadIdx.x == 0) sig_wait(sig);
    __syncthreads();
  }
  combine_bwd_rows<T, NVL, PEER>(dY, Recv, tok_of, kept, gate, k, d, E, C, c0, nc, Cm, El, P, me, dSend, peer, dg);
  if constexpr (PEER) {
    __syncthreads();
    if (threadIdx.x == 0) sig_post_last(sig);  // the last CTA: READY of the backward dispatch
  }
}

// Split dispatch (n = 1, fused transport): the owner blocks of the send layout
// (owner o = experts [o*El, (o+1)*El), El*Cm rows each) in the order j = j0 .. j0+nj-1,
// owner(j) = (me - j) mod P — j = 0 is this rank's own block (no NVLink), then the peers
// in descending order, so at step j every rank s writes to s - j (no incast) and rank o
// receives first from o + 1, then o + 2, ... (the order its expert GEMM consumes them in,
// gemm_tc.cu `src_wait`).  All CTAs of the (persistent) grid walk the blocks in that
// order; the last CTA done with block j posts READY to owner(j) alone (done[j]), so an
// owner's GEMM starts on a source's rows as soon as they are in.
// BWD = false: the permute (S3 + S4); BWD = true: combine-backward (S8a; dg too).
template <typename T, int NVL, bool BWD>
__global__ void __launch_bounds__(256) split_rows_kernel(const T* __restrict__ src, const T* __restrict__ Recv,
                                                         const int* __restrict__ tok_of,
                                                         const int* __restrict__ kept,
                                                         const float* __restrict__ gate, int k, int d, int E, int C,
                                                         int Cm, int El, int P, int me, int j0, int nj,
                                                         T* const* __restrict__ peer, float* __restrict__ dg,
                                                         PeerSignal sig, unsigned int* __restrict__ done) {
  pdl_enter();
  if (sig.wait) {  // (backward: the owners' dO is free)
    if (threadIdx.x == 0) sig_wait(sig);
    __syncthreads();
  }
  constexpr int R = BWD ? combine_bwd_R<NVL>() : permute_R<NVL>();
  const long long blk = (long long)El * Cm;
  const long long wpc = blockDim.x >> 5;
  const long long gw = (long long)blockIdx.x * wpc + (threadIdx.x >> 5);
  const long long nw = (long long)gridDim.x * wpc;
  for (int j = j0; j < j0 + nj; ++j) {
    const int owner = ((me - j) % P + P) % P;
    const long long base = (long long)owner * blk, end = base + blk;
    for (long long r0 = base + gw * R; r0 < end; r0 += nw * R) {
      if constexpr (BWD)
        combine_bwd_rows_at<T, NVL, true>(src, Recv, tok_of, kept, gate, k, d, E, C, 0, r0, end, Cm, El, P, me,
                                          nullptr, peer, dg);
      else
        permute_rows_at<T, NVL, true>(src, tok_of, kept, k, d, E, C, 0, r0, end, Cm, El, P, me, nullptr, peer);
    }
    if (j > 0 && sig.post) {
      __syncthreads();
      if (threadIdx.x == 0) sig_post_owner_last(sig, done + j, owner, gridDim.x);
    }
  }
}

// This rank's per-expert counts into every owner's recv_kept (after their FREE), then
// COUNT posted: the owners' tile lists need every source's counts, the rows may follow.
__global__ void dispatch_counts_kernel(const int* __restrict__ kept, int P, int El, int me,
                                       int* const* __restrict__ peer_counts, PeerSignal free_sig,
                                       PeerSignal count_sig) {
  pdl_enter();
  if (threadIdx.x == 0) sig_wait(free_sig);
  __syncthreads();
  for (int i = threadIdx.x; i < P * El; i += blockDim.x) peer_counts[i / El][me * El + i % El] = kept[i];
  __syncthreads();
  if (threadIdx.x == 0) sig_post(count_sig);
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

// vectors per lane per row, rounded up to an instantiated width (0 = strided loop)
inline int nvl_of(int d, int dtype) {
  const int nv = d / (dtype == 0 ? 4 : 8);
  const int need = (nv + 31) / 32;
  if (need <= 4) return need < 1 ? 1 : need;
  if (need <= 6) return 6;
  if (need <= 8) return 8;
  return 0;
}

// rows handled by one warp for a given NVL (must match the kernels' R)
inline int rows_per_warp(int nvl, int loads_per_row) {
  if (nvl == 0) return 1;
  const int per = nvl * loads_per_row;
  return per >= kLoadsPerLane ? 1 : kLoadsPerLane / per;
}

#define LINA_DISPATCH_NVL(nvl, ...)             \
  do {                                          \
    switch (nvl) {                              \
      case 1: { constexpr int NV_ = 1; __VA_ARGS__; } break; \
      case 2: { constexpr int NV_ = 2; __VA_ARGS__; } break; \
      case 3: { constexpr int NV_ = 3; __VA_ARGS__; } break; \
      case 4: { constexpr int NV_ = 4; __VA_ARGS__; } break; \
      case 6: { constexpr int NV_ = 6; __VA_ARGS__; } break; \
      case 8: { constexpr int NV_ = 8; __VA_ARGS__; } break; \
      default: { constexpr int NV_ = 0; __VA_ARGS__; } break; \
    }                                           \
  } while (0)

template <bool PEER>
static void permute_any(int dtype, const void* X, const int* tok_of, int k, int d, int E, int C, int c0, int nc,
                        int Cm, int El, int P, int me, void* Send, void* const* peer, const int* kept,
                        void* const* peer_counts, const PeerSignal& sig, cudaStream_t s) {
  const long long rows = (long long)nc * E * Cm;
  if (rows == 0 && !PEER) return;
  const int nvl = nvl_of(d, dtype);
  const long long warps = std::max(1LL, (rows + rows_per_warp(nvl, 1) - 1) / rows_per_warp(nvl, 1));
  LINA_DISPATCH_T(dtype, LINA_DISPATCH_NVL(nvl, launch_k(permute_kernel<ET, NV_, PEER>, dim3(blocks_for_warps(warps)),
                             dim3(256), 0, s, (const ET*)X, tok_of, k, d, E, C, c0, nc, Cm, El, P, me, (ET*)Send,
                             (ET* const*)peer, kept, (int* const*)peer_counts, sig)));
  LINA_LAUNCH_CHECK();
}

void launch_permute(int dtype, const void* X, const int* tok_of, const int* kept, int k, int d, int E, int C,
                    int n, int Cm, void* Send, cudaStream_t s) {
  permute_any<false>(dtype, X, tok_of, k, d, E, C, 0, n, Cm, 0, 1, 0, Send, nullptr, kept, nullptr, PeerSignal{},
                     s);
}

void launch_combine(int dtype, const void* Recv, const int* idx, const int* slot, const float* gate,
                    int T, int k, int d, int E, int C, int n, int Cm, void* Y, cudaStream_t s,
                    const PeerSignal* sig, const int* ebase) {
  const PeerSignal sg = sig ? *sig : PeerSignal{};
  if (T <= 0 && !sig) return;
  const int nvl = nvl_of(d, dtype);
  const int U = nvl > 0 ? kLoadsPerLane / nvl : 0;
  if (nvl > 0 && (k == 1 || k == 2) && U >= 1) {
    const int tp = U / k > 0 ? U / k : 1;
    const long long warps = std::max(1LL, ((long long)T + tp - 1) / tp);
    if (k == 1)
      LINA_DISPATCH_T(dtype, LINA_DISPATCH_NVL(nvl, launch_k(combine_kernel<ET, NV_, 1>, dim3(blocks_for_warps(warps)),
                                 dim3(256), 0, s, (const ET*)Recv, idx, slot, gate, T, k, d, E, C, n, Cm, (ET*)Y, sg, ebase)));
    else
      LINA_DISPATCH_T(dtype, LINA_DISPATCH_NVL(nvl, launch_k(combine_kernel<ET, NV_, 2>, dim3(blocks_for_warps(warps)),
                                 dim3(256), 0, s, (const ET*)Recv, idx, slot, gate, T, k, d, E, C, n, Cm, (ET*)Y, sg, ebase)));
  } else {
    LINA_DISPATCH_T(dtype, launch_k(combine_loop_kernel<ET>, dim3(blocks_for_warps(std::max(1, T))), dim3(256), 0, s,
                                    (const ET*)Recv, idx, slot, gate, T, k, d, E, C, n, Cm, (ET*)Y, sg, ebase));
  }
  LINA_LAUNCH_CHECK();
}

template <bool PEER>
static void combine_bwd_any(int dtype, const void* dY, const void* Recv, const int* tok_of, const int* kept,
                            const float* gate, int T, int k, int d, int E, int C, int c0, int nc, int Cm, int El,
                            int P, int me, void* dSend, void* const* peer, float* dg, const PeerSignal& sig,
                            cudaStream_t s) {
  // dg = 0 for dropped assignments: zeroed once, before the first chunk range
  if (T > 0 && c0 == 0) LINA_CUDA_CHECK(cudaMemsetAsync(dg, 0, sizeof(float) * (size_t)T * k, s));
  const long long rows = (long long)nc * E * Cm;
  if (rows == 0 && !PEER) return;
  const int nvl = nvl_of(d, dtype);
  const long long warps = std::max(1LL, (rows + rows_per_warp(nvl, 2) - 1) / rows_per_warp(nvl, 2));
  LINA_DISPATCH_T(dtype, LINA_DISPATCH_NVL(nvl, launch_k(combine_bwd_kernel<ET, NV_, PEER>,
                             dim3(blocks_for_warps(warps)), dim3(256), 0, s, (const ET*)dY, (const ET*)Recv, tok_of,
                             kept, gate, k, d, E, C, c0, nc, Cm, El, P, me, (ET*)dSend, (ET* const*)peer, dg, sig)));
  LINA_LAUNCH_CHECK();
}

void launch_combine_bwd(int dtype, const void* dY, const void* Recv, const int* tok_of, const int* kept,
                        const float* gate, int T, int k, int d, int E, int C, int n, int Cm,
                        void* dSend, float* dg, cudaStream_t s) {
  combine_bwd_any<false>(dtype, dY, Recv, tok_of, kept, gate, T, k, d, E, C, 0, n, Cm, 0, 1, 0, dSend, nullptr, dg,
                         PeerSignal{}, s);
}

void launch_permute_peer(int dtype, const void* X, const int* tok_of, const int* kept, int k, int d, int E,
                         int C, int c0, int nc, int Cm, int El, int P, int me, void* const* peer_rows,
                         void* const* peer_counts, const PeerSignal& sig, cudaStream_t s) {
  permute_any<true>(dtype, X, tok_of, k, d, E, C, c0, nc, Cm, El, P, me, nullptr, peer_rows, kept, peer_counts, sig,
                    s);
}

void launch_combine_bwd_peer(int dtype, const void* dY, const void* Recv, const int* tok_of, const int* kept,
                             const float* gate, int T, int k, int d, int E, int C, int c0, int nc, int Cm, int El,
                             int P, int me, void* const* peer_rows, float* dg, const PeerSignal& sig,
                             cudaStream_t s) {
  combine_bwd_any<true>(dtype, dY, Recv, tok_of, kept, gate, T, k, d, E, C, c0, nc, Cm, El, P, me, nullptr,
                        peer_rows, dg, sig, s);
}

void launch_dispatch_counts(const int* kept, int P, int El, int me, void* const* peer_counts,
                            const PeerSignal& free_sig, const PeerSignal& count_sig, cudaStream_t s) {
  launch_k(dispatch_counts_kernel, dim3(1), dim3(256), 0, s, kept, P, El, me, (int* const*)peer_counts, free_sig,
           count_sig);
  LINA_LAUNCH_CHECK();
}

template <bool BWD>
static void split_any(int dtype, const void* src, const void* Recv, const int* tok_of, const int* kept,
                      const float* gate, int k, int d, int E, int C, int Cm, int El, int P, int me,
                      void* const* peer_rows, float* dg, int j0, int nj, int grid, const PeerSignal& sig,
                      unsigned int* done, cudaStream_t s) {
  const int nvl = nvl_of(d, dtype);
  // persistent grids (the peers' rows beside the expert GEMM) use 128-thread CTAs: one fits
  // next to a GEMM CTA in the SM's registers (<= 64K - 320 x 136) and its 1 KB of reserved
  // shared memory next to the GEMM's 225.5 KB
  int threads = 128;
  if (grid <= 0) {  // one pass over one block
    const long long rows = (long long)El * Cm * nj;
    const int r = rows_per_warp(nvl, BWD ? 2 : 1);
    threads = 256;
    grid = blocks_for_warps(std::max(1LL, (rows + r - 1) / r));
  }
  LINA_DISPATCH_T(dtype, LINA_DISPATCH_NVL(nvl, launch_k(split_rows_kernel<ET, NV_, BWD>, dim3(grid), dim3(threads), 0, s,
                             (const ET*)src, (const ET*)Recv, tok_of, kept, gate, k, d, E, C, Cm, El, P, me, j0, nj,
                             (ET* const*)peer_rows, dg, sig, done)));
  LINA_LAUNCH_CHECK();
}

void launch_permute_split(int dtype, const void* X, const int* tok_of, const int* kept, int k, int d, int E, int C,
                          int Cm, int El, int P, int me, void* const* peer_rows, int j0, int nj, int grid,
                          const PeerSignal& sig, unsigned int* done, cudaStream_t s) {
  split_any<false>(dtype, X, nullptr, tok_of, kept, nullptr, k, d, E, C, Cm, El, P, me, peer_rows, nullptr, j0, nj,
                   grid, sig, done, s);
}

void launch_combine_bwd_split(int dtype, const void* dY, const void* Recv, const int* tok_of, const int* kept,
                              const float* gate, int k, int d, int E, int C, int Cm, int El, int P, int me,
                              void* const* peer_rows, float* dg, int j0, int nj, int grid, const PeerSignal& sig,
                              unsigned int* done, cudaStream_t s) {
  split_any<true>(dtype, dY, Recv, tok_of, kept, gate, k, d, E, C, Cm, El, P, me, peer_rows, dg, j0, nj, grid, sig,
                  done, s);
}

}  // namespace lina
