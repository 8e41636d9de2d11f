// Stand-alone all-to-all movers of the fused transport (instrumentation: the
// collectives-only pass of lina_profile_enable flag 4, SURVEY.md §8(d) T_a2a(n)).
//
// In the real pass the combine all-to-all is the GEMM2 / dgrad2 epilogue's peer stores
// (gemm_tc.cu); to time the exchange alone, this kernel moves the same rows — the valid
// rows of every segment (c, s, el) of micro-op c in the receive layout [n][P][El][Cm][d]
// — into the owner s's send-layout buffer at segment c*E + me*El + el (the
// return all-to-all), by 16-byte NVLink peer stores, and posts READY of micro-op c from
// its last CTA, exactly as the epilogue does.
#include <cuda_bf16.h>

#include <algorithm>

#include "../common.h"
#include "../kernels.h"

namespace lina {
namespace {

// grid (x, P*El): blockIdx.y = segment (s, el) of chunk c; 8 warps stride its rows
__global__ void __launch_bounds__(256) push_segments_kernel(const uint4* __restrict__ src, uint4* const* __restrict__ peer,
                                                            const int* __restrict__ vcount, int c, int P, int El, int E,
                                                            int Cm, int me, int nv, PeerSignal sig) {
  pdl_enter();
  const int seg = blockIdx.y;  // s * El + el
  const int s = seg / El, el = seg % El;
  const int gseg = c * P * El + seg;
  const int rows = vcount[gseg];
  const uint4* from = src + (size_t)gseg * Cm * nv;
  uint4* to = peer[s] + ((size_t)c * E + (size_t)me * El + el) * Cm * nv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = blockIdx.x * 8 + warp; r < rows; r += gridDim.x * 8) {
    const uint4* a = from + (size_t)r * nv;
    uint4* b = to + (size_t)r * nv;
    for (int v = lane; v < nv; v += 32) b[v] = a[v];
  }
  __syncthreads();
  if (threadIdx.x == 0) sig_post_last(sig);
}

}  // namespace

void launch_push_segments(int dtype, const void* recv_layout, void* const* peer_send_layout, const int* vcount,
                          int c, int P, int El, int E, int Cm, int me, int d, const PeerSignal& sig, cudaStream_t s) {
  const int elt = dtype == 1 ? 2 : 4;
  const int nv = d * elt / 16;
  dim3 grid(std::max(1, std::min(32, (Cm + 7) / 8)), P * El);
  launch_k(push_segments_kernel, grid, dim3(256), 0, s, (const uint4*)recv_layout, (uint4* const*)peer_send_layout,
           vcount, c, P, El, E, Cm, me, nv, sig);
  LINA_LAUNCH_CHECK();
}

}  // namespace lina
