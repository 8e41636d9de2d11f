// Shared device/host helpers for the Lina B200 library (internal header).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <string>
#include <utility>

namespace lina {

// ---------------------------------------------------------------- error plumbing
void set_error(const std::string& msg);           // thread-local message (api.cpp)

struct CudaError {
  std::string what;
};

#define LINA_CUDA_CHECK(expr)                                                              \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      throw ::lina::CudaError{std::string(#expr) + " -> " + cudaGetErrorString(_e) + " (" + \
                              __FILE__ + ":" + std::to_string(__LINE__) + ")"};            \
  } while (0)

// Process-wide count of this library's kernel launches (lina_profile_read).
void count_launch();
#define LINA_LAUNCH_CHECK()                   \
  do {                                        \
    ::lina::count_launch();                   \
    LINA_CUDA_CHECK(cudaGetLastError());      \
  } while (0)

// ---------------------------------------------------------------- programmatic dependent launch
// Kernels of the layer are launched with programmatic stream serialization: a kernel may
// be scheduled while its predecessor on the stream drains.  Every such kernel waits for
// its predecessor's completion (and memory) before touching global memory
// (griddepcontrol.wait), then lets its own successor be scheduled (launch_dependents).
// No-ops when the kernel was launched without the attribute.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}
#endif
bool pdl_enabled();  // LINA_PDL=0 disables (api.cpp)

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  LINA_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// ---------------------------------------------------------------- dtype traits
template <typename T> struct Elt;
template <> struct Elt<float> {
  __device__ __forceinline__ static float to_f(float x) { return x; }
  __device__ __forceinline__ static float from_f(float x) { return x; }
};
template <> struct Elt<__nv_bfloat16> {
  __device__ __forceinline__ static float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  __device__ __forceinline__ static __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
};

// 16-byte vector of T (8 bf16 or 4 fp32)
template <typename T> struct Vec16 {
  static constexpr int N = 16 / sizeof(T);
};

__device__ __forceinline__ void load16(const void* p, float* out, const float*) {
  float4 v = *reinterpret_cast<const float4*>(p);
  out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
}
__device__ __forceinline__ void load16(const void* p, float* out, const __nv_bfloat16*) {
  uint4 v = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    out[2 * i] = f.x; out[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void store16(void* p, const float* in, float*) {
  *reinterpret_cast<float4*>(p) = make_float4(in[0], in[1], in[2], in[3]);
}
__device__ __forceinline__ void store16(void* p, const float* in, __nv_bfloat16*) {
  uint4 v;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(in[2 * i], in[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = v;
}

// ---------------------------------------------------------------- chunk geometry (R10)
// The n all-to-all micro-ops split the capacity slots of every expert along the token
// dimension ("partition the data in the token dimension"): chunk c covers slots
// [c*Cm, min((c+1)*Cm, C)) with pitch Cm = ceil(C/n) rounded up to a multiple of the
// tensor-core tile height (256, else 128, else 64 rows) whenever all n chunks stay
// non-empty, so chunk boundaries do not cut expert GEMM tiles.  Results do not depend
// on n (the oracle has no chunks); only the last chunk can be shorter.
__host__ __device__ __forceinline__ int chunk_pitch(int C, int n) {
  if (n <= 1) return C;
  const int base = (C + n - 1) / n;
  for (int a = 256; a >= 64; a >>= 1) {
    const int cm = (base + a - 1) / a * a;
    if ((long long)(n - 1) * cm < C) return cm;
  }
  return base;
}
__host__ __device__ __forceinline__ int chunk_begin(int c, int C, int n) {
  const long long b = (long long)c * chunk_pitch(C, n);
  return b < C ? (int)b : C;
}
// The chunk holding slot s.
__host__ __device__ __forceinline__ int chunk_of(int s, int C, int n) { return s / chunk_pitch(C, n); }
__host__ __device__ __forceinline__ int chunk_rows_max(int C, int n) { return chunk_pitch(C, n); }
// Row of (expert e, capacity slot s) in the chunk-major send layout [n][E][Cm][w]
// (Cm = chunk_pitch(C, n), precomputed by the host: one division per call).
__host__ __device__ __forceinline__ size_t send_row(int e, int s, int E, int C, int n, int Cm) {
  (void)C;
  (void)n;
  const int c = s / Cm;
  return ((size_t)c * E + e) * Cm + (s - c * Cm);
}
// First slot of chunk c given the pitch.
__host__ __device__ __forceinline__ int chunk_begin_p(int c, int C, int Cm) {
  const long long b = (long long)c * Cm;
  return b < C ? (int)b : C;
}

}  // namespace lina
