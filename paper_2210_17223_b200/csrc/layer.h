// Internal entry points between api.cpp, layer.cpp, infer.cpp and sched.cpp.
#pragma once
#include "internal.h"
#include "kernels.h"

namespace lina {

void moe_forward(lina_comm* cm, const Plan& p, const void* tokens, const float* gate_w,
                 const void* w1, const void* w2, void* out, void* saved, void* ws,
                 lina_route* route, cudaStream_t s);
void moe_backward(lina_comm* cm, const Plan& p, const void* saved, const void* dout,
                  const void* tokens, const float* gate_w, const void* w1, const void* w2,
                  void* dtokens, float* dgate_w, void* dw1, void* dw2, void* ws, cudaStream_t s);

// Expert GEMM dispatch: tcgen05 kernels for bf16 (when shapes allow), SIMT otherwise.
void launch_expert_row_gemm(int dtype, const RowGemm& g, bool b_kmajor, int epi, cudaStream_t s);
void launch_expert_wgrad(int dtype, const WGrad& g, cudaStream_t s);
// Force the SIMT path for bf16 too (tests/benchmarks of the reference GEMM).
void set_force_simt(bool on);

// Scheduler hooks called by the layer (sched.cpp).
void sched_a2a_imminent(lina_comm* cm);                   // combine-bwd started
void sched_a2a_begin(lina_comm* cm, cudaStream_t a2a_stream);
void sched_a2a_end(lina_comm* cm, cudaStream_t a2a_stream);  // phase ends there

Scheduler* sched_create(lina_comm* cm);
void sched_destroy(Scheduler* s);
void sched_config(Scheduler* s, lina_policy p, size_t partition_bytes);
void sched_submit(Scheduler* s, void* grad, size_t count, lina_dtype dt, cudaStream_t ready);
void sched_wait(Scheduler* s, cudaStream_t st);
void sched_stats(Scheduler* s, int64_t* issued, int64_t* deferred);

// Placement (placement.cpp).
lina_status placement_compute(const double* pop, int E, int N, int mpd, lina_placement* out,
                              std::string* err);
void replica_split(int count, int replicas, int source_rank, int* out);

}  // namespace lina
