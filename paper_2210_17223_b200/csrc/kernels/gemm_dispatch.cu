// Expert GEMM dispatch: tcgen05 (gemm_tc.cu) for bf16 when the shapes allow it,
// the SIMT kernels (gemm_simt.cu) otherwise.
#include "../common.h"
#include "../kernels.h"
#include "../layer.h"

namespace lina {

static bool g_force_simt = false;
void set_force_simt(bool on) { g_force_simt = on; }

void launch_expert_row_gemm(int dtype, const RowGemm& g, bool b_kmajor, int epi, cudaStream_t s) {
  launch_row_gemm_simt(dtype, g, b_kmajor, epi, s);
}

void launch_expert_wgrad(int dtype, const WGrad& g, cudaStream_t s) {
  launch_wgrad_simt(dtype, g, s);
}

}  // namespace lina
