"""TMA bulk-tensor store bandwidth, local vs NVLink peer (diagnostic).

One CTA per SM, 4 warps; each warp stores 32 x 64 bf16 boxes (4 KB, 128B swizzle) from
shared memory to a [rows][N] bf16 tensor through a tensor map with `depth` bulk groups
in flight (cp.async.bulk.wait_group.read).  Device-timed.  Needs 2 GPUs.
    python tools/p2p_tma_bw.py"""
import json

import torch
from torch.utils.cpp_extension import load_inline

SRC = r"""
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdexcept>
#include <cstdint>

template <int DEPTH>
__global__ void __launch_bounds__(128) tma_store_kernel(const __grid_constant__ CUtensorMap m, int rows, int N,
                                                        int iters) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* box = sm + warp * DEPTH * 4096;
  for (int i = lane; i < DEPTH * 4096 / 16; i += 32) reinterpret_cast<uint4*>(box)[i] = make_uint4(i, 1, 2, 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane != 0) return;
  const int nbx = N / 64, nby = rows / 32;
  const int gw = blockIdx.x * 4 + warp, nw = gridDim.x * 4;
  int k = 0;
  for (int it = 0; it < iters; ++it)
    for (int t = gw; t < nbx * nby; t += nw, ++k) {
      const int x = (t % nbx) * 64, y = (t / nbx) * 32;
      const unsigned char* src = box + (k % DEPTH) * 4096;
      if (k >= DEPTH) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(DEPTH - 1) : "memory");
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&m),
                   "r"((unsigned)__cvta_generic_to_shared(src)), "r"(x), "r"(y) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

void enable_peer(int a, int b) {
  cudaSetDevice(a);
  cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
  if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) throw std::runtime_error(cudaGetErrorString(e));
  cudaGetLastError();
}

void run(long long dst, int rows, int N, int depth, int blocks, int iters, long long stream) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)N * 2};
  cuuint32_t box[2] = {64, 32}, es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)dst, dims, str, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("encode failed");
  const int smem = 4 * depth * 4096 + 1024;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<blocks, 128, smem, (cudaStream_t)stream>>>(m, rows, N, iters);
  };
  if (depth == 1) go(tma_store_kernel<1>);
  else if (depth == 2) go(tma_store_kernel<2>);
  else if (depth == 4) go(tma_store_kernel<4>);
  else go(tma_store_kernel<8>);
}
"""
CPP = "void enable_peer(int a, int b); void run(long long dst, int rows, int N, int depth, int blocks, int iters, long long stream);"
ext = load_inline("p2p_tma_bw", cpp_sources=CPP, cuda_sources=SRC, functions=["enable_peer", "run"],
                  extra_cuda_cflags=["-O3", "-gencode", "arch=compute_100a,code=sm_100a"],
                  extra_ldflags=["-lcuda"], verbose=False)
ext.enable_peer(0, 1)
ext.enable_peer(1, 0)
rows, N = 16384, 768  # 24 MB
dst = {g: torch.empty(rows * N, dtype=torch.bfloat16, device=f"cuda:{g}") for g in (0, 1)}


def timed(pairs, depth, blocks=148, iters=4):
    for dev, buf in pairs:
        with torch.cuda.device(dev):
            ext.run(buf.data_ptr(), rows, N, depth, blocks, 1, torch.cuda.current_stream().cuda_stream)
    for dev, _ in pairs:
        torch.cuda.synchronize(dev)
    evs = []
    for dev, buf in pairs:
        with torch.cuda.device(dev):
            st = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            ext.run(buf.data_ptr(), rows, N, depth, blocks, iters, st.cuda_stream)
            e1.record(st)
            evs.append((dev, e0, e1))
    out = []
    for dev, e0, e1 in evs:
        torch.cuda.synchronize(dev)
        out.append(round(rows * N * 2 * iters / (e0.elapsed_time(e1) / 1e3) / 1e9, 1))
    return out


for depth in (1, 2, 4, 8):
    print(json.dumps({"depth": depth, "local_GBps": timed([(0, dst[0])], depth),
                      "peer_GBps": timed([(0, dst[1])], depth),
                      "peer_both_GBps": timed([(0, dst[1]), (1, dst[0])], depth)}), flush=True)
