// S5 / S8c expert FFN GEMMs on CUDA cores (fp32 path; also the bf16 reference path).
//
// "Every expert is a fully-connected two-layer network using ReLU".
// fp32 tokens use this path forever: TF32 tensor cores cannot meet the 1e-5
// tolerance (north_star).  The bf16 production path is gemm_tc.cu (tcgen05).
//
// Row-grouped GEMM (forward GEMM1/GEMM2, backward dgrad):
//   for every segment g of a chunk (one (source rank, local expert) pair, Cm rows,
//   vcount[g] of them valid):  D[rows] = epi(A[rows] · Bᵀ_e)
//   A [rows][K] K-major; B_e either K-major ([N][K], nn.Linear weight) or
//   MN-major ([K][N], the transposed use of the other weight in dgrad).
// Weight-gradient GEMM (wgrad): D_e[M][N] = Σ_{segments of e} Σ_{valid rows} A_rᵀ B_r.
// 64x64 CTA tiles, BK=16, 256 threads with 4x4 register micro-tiles; each output
// is one fp32 FMA chain in ascending K (deterministic, no split-K).
#include "../common.h"
#include "../kernels.h"

namespace lina {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;

template <typename T, bool B_KMAJOR, int EPI>
__global__ void __launch_bounds__(256) row_gemm_kernel(RowGemm p) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int mtiles = (p.Cm + BM - 1) / BM;
  const int gi = blockIdx.x / mtiles;
  const int m0 = (blockIdx.x % mtiles) * BM;
  const int seg = p.seg0 + gi;
  const int v = p.vcount[seg];
  if (m0 >= v) return;
  const int n0 = blockIdx.y * BN;
  const int el = p.seg_expert ? p.seg_expert[gi % p.El] : gi % p.El;
  const T* A = (const T*)p.A + (size_t)seg * p.Cm * p.K;
  const T* B = (const T*)p.B + (size_t)el * p.N * p.K;
  const int ty = tid / 16, tx = tid % 16;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < p.K; k0 += BK) {
    {
      const int r = tid / 4, kq = (tid % 4) * 4;
      const int m = m0 + r;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int kk = k0 + kq + i;
        As[kq + i][r] = (m < v && kk < p.K) ? Elt<T>::to_f(A[(size_t)m * p.K + kk]) : 0.f;
      }
    }
    if (B_KMAJOR) {
      const int r = tid / 4, kq = (tid % 4) * 4;
      const int nn = n0 + r;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int kk = k0 + kq + i;
        Bs[kq + i][r] = (nn < p.N && kk < p.K) ? Elt<T>::to_f(B[(size_t)nn * p.K + kk]) : 0.f;
      }
    } else {
      const int kr = tid / 16, nq = (tid % 16) * 4;
      const int kk = k0 + kr;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int nn = n0 + nq + i;
        Bs[kr][nq + i] = (nn < p.N && kk < p.K) ? Elt<T>::to_f(B[(size_t)kk * p.N + nn]) : 0.f;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  T* D = (T*)p.D + (size_t)seg * p.Cm * p.N;
  const T* aux = (const T*)p.aux + (size_t)seg * p.Cm * p.N;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= p.Cm) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int nn = n0 + tx * 4 + j;
      if (nn >= p.N) continue;
      float x = acc[i][j];
      if (EPI == kEpiRelu) x = fmaxf(x, 0.f);
      if (EPI == kEpiMask) x = (Elt<T>::to_f(aux[(size_t)m * p.N + nn]) > 0.f) ? x : 0.f;
      D[(size_t)m * p.N + nn] = Elt<T>::from_f(x);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) wgrad_kernel(WGrad p) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN, el = blockIdx.z;
  const int ty = tid / 16, tx = tid % 16;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  // segments of expert el: (c*P + s)*El + el, or the dropless range
  const int nlist = p.seg_range ? p.seg_range[2 * el + 1] - p.seg_range[2 * el] : p.nchunks * p.P;
  for (int li = 0; li < nlist; ++li) {
    {
      const int seg = p.seg_range ? p.seg_range[2 * el] + li : li * p.El + el;
      const int v = p.vcount[seg];
      const T* A = (const T*)p.A + (size_t)seg * p.Cm * p.M;
      const T* B = (const T*)p.B + (size_t)seg * p.Cm * p.N;
      for (int r0 = 0; r0 < v; r0 += BK) {
        {
          const int kr = tid / 16, q = (tid % 16) * 4;
          const int r = r0 + kr;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int m = m0 + q + i, nn = n0 + q + i;
            As[kr][q + i] = (r < v && m < p.M) ? Elt<T>::to_f(A[(size_t)r * p.M + m]) : 0.f;
            Bs[kr][q + i] = (r < v && nn < p.N) ? Elt<T>::to_f(B[(size_t)r * p.N + nn]) : 0.f;
          }
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
          float a[4], b[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
          for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
      }
    }
  }
  T* D = (T*)p.D + (size_t)el * p.M * p.N;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int nn = n0 + tx * 4 + j;
      if (nn < p.N) D[(size_t)m * p.N + nn] = Elt<T>::from_f(acc[i][j]);
    }
  }
}

template <typename T>
void launch_row_t(const RowGemm& p, bool b_kmajor, int epi, cudaStream_t s) {
  dim3 grid(p.nseg * ((p.Cm + BM - 1) / BM), (p.N + BN - 1) / BN);
  if (b_kmajor) {
    if (epi == kEpiRelu) row_gemm_kernel<T, true, kEpiRelu><<<grid, 256, 0, s>>>(p);
    else if (epi == kEpiMask) row_gemm_kernel<T, true, kEpiMask><<<grid, 256, 0, s>>>(p);
    else row_gemm_kernel<T, true, kEpiNone><<<grid, 256, 0, s>>>(p);
  } else {
    if (epi == kEpiRelu) row_gemm_kernel<T, false, kEpiRelu><<<grid, 256, 0, s>>>(p);
    else if (epi == kEpiMask) row_gemm_kernel<T, false, kEpiMask><<<grid, 256, 0, s>>>(p);
    else row_gemm_kernel<T, false, kEpiNone><<<grid, 256, 0, s>>>(p);
  }
}

}  // namespace

void launch_row_gemm_simt(int dtype, const RowGemm& p, bool b_kmajor, int epi, cudaStream_t s) {
  if (p.nseg <= 0 || p.Cm <= 0) return;
  if (dtype == 0) launch_row_t<float>(p, b_kmajor, epi, s);
  else launch_row_t<__nv_bfloat16>(p, b_kmajor, epi, s);
  LINA_LAUNCH_CHECK();
}

void launch_wgrad_simt(int dtype, const WGrad& p, cudaStream_t s) {
  dim3 grid((p.M + BM - 1) / BM, (p.N + BN - 1) / BN, p.El);
  if (p.El <= 0) return;
  if (dtype == 0) wgrad_kernel<float><<<grid, 256, 0, s>>>(p);
  else wgrad_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(p);
  LINA_LAUNCH_CHECK();
}

}  // namespace lina
