// Expert GEMM dispatch: tcgen05 (gemm_tc.cu) for bf16 when the shapes allow it,
// the SIMT kernels (gemm_simt.cu) otherwise.
#include <stdlib.h>

#include "../common.h"
#include "../kernels.h"
#include "../layer.h"

namespace lina {

// LINA_FORCE_SIMT=1 routes bf16 through the CUDA-core kernels (reference path for tests/benchmarks).
static bool g_force_simt = [] {
  const char* e = getenv("LINA_FORCE_SIMT");
  return e && e[0] == '1';
}();
void set_force_simt(bool on) { g_force_simt = on; }

void launch_expert_row_gemm(int dtype, const RowGemm& g, bool b_kmajor, int epi, cudaStream_t s) {
  if (dtype == 1 && !g_force_simt && tc_row_supported(g)) {
    launch_row_gemm_tc(g, b_kmajor, epi, s);
  } else {
    if (g.sig) throw CudaError{"in-kernel peer signals need the tcgen05 GEMM (unset LINA_FORCE_SIMT)"};
    launch_row_gemm_simt(dtype, g, b_kmajor, epi, s);
  }
}

void launch_expert_wgrad(int dtype, const WGrad& g, cudaStream_t s) {
  if (dtype == 1 && !g_force_simt && tc_wgrad_supported(g)) launch_wgrad_tc(g, s);
  else launch_wgrad_simt(dtype, g, s);
}

}  // namespace lina
