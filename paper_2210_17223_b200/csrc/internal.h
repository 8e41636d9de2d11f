// Internal host-side types of the Lina B200 library.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <condition_variable>
#include <deque>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/lina.h"
#include "common.h"

namespace lina {

struct NcclError {
  std::string what;
};
struct ArgError {
  std::string what;
};
struct StatusError {
  lina_status status;
  std::string what;
};

#define LINA_NCCL_CHECK(expr)                                                                  \
  do {                                                                                         \
    ncclResult_t _r = (expr);                                                                  \
    if (_r != ncclSuccess)                                                                     \
      throw ::lina::NcclError{std::string(#expr) + " -> " + ncclGetErrorString(_r) + " (" +    \
                              __FILE__ + ":" + std::to_string(__LINE__) + ")"};                \
  } while (0)

class Scheduler;    // sched.cpp
class CeTransport;  // ce.cpp

// Buffer plan for one descriptor on one communicator (layer.cpp).
struct Plan {
  int T, d, f, E, k, C, n, P, El, Cm, dt;  // dt = element bytes
  int tile_rows;                           // expert row-GEMM M tile (128 or 256)
  bool bf16;
  // offsets (bytes) into `saved`
  size_t s_probs, s_idx, s_gate, s_slot, s_kept, s_tokof, s_recvkept, s_vcount, s_mtp, s_R, s_H,
      s_C, s_mask;
  size_t s_mtpt = 0, s_rbase = 0;  // tail-split tile lists (tc row GEMMs with 256-row tiles)
  bool tail_split = false;
  bool half_tails = false;                 // RowGemm::half_tails (LINA_HALF128, layer.cpp)
  size_t saved_bytes;
  // offsets into `workspace`
  size_t w_route, w_D, w_O, w_dg, w_dwg, w_dS, w_dO, w_dH, w_dXe, w_dXs;
  size_t ws_bytes;
  uint64_t peer_key;  // hash of the peer-visible geometry (checked across ranks on first mapping)
  // dropless layout (capacity == 0; §8(f) row 4): V virtual segments of tile_rows rows per
  // receive buffer, T·k compact rows per source buffer, the count table and the layout tables
  bool dropless = false;  // the variable layout (capacity 0 and / or pack > 1)
  int pack = 1;           // expert packing factor m (El = m·E/P experts hosted per rank)
  int V = 0;
  size_t s_allc = 0, s_tab = 0;
  size_t rows_send() const { return (size_t)n * E * Cm; }
  size_t rows_recv() const { return (size_t)n * P * El * Cm; }
};

Plan make_plan(const lina_moe_desc& desc, int world);

}  // namespace lina

namespace lina {
struct Trace;
}

struct lina_comm {
  int rank = 0, world = 1, device = 0, num_sms = 148;
  unsigned int* tile_ctr = nullptr;  // expert-GEMM dynamic tile counter (LINA_GEMM_DYN; self-resetting)
  ncclComm_t ep_disp = nullptr;  // dispatch-direction all-to-all micro-ops
  ncclComm_t ep_comb = nullptr;  // combine-direction all-to-all micro-ops (full-duplex, H8)
  ncclComm_t dp = nullptr;       // non-expert gradient allreduce micro-ops
  cudaStream_t hi = nullptr;     // dispatch a2a (greatest priority)
  cudaStream_t hi2 = nullptr;    // combine a2a (greatest priority)
  cudaStream_t lo = nullptr;     // allreduce micro-ops (least priority)
  std::vector<cudaEvent_t> ev;   // event pool (timing disabled)
  lina::Scheduler* sched = nullptr;
  lina::CeTransport* ce = nullptr;  // peer mappings + flags (NULL = NCCL all-to-all only)
  int transport = 0;                // 0 NCCL, 1 copy engines, 2 fused into the kernels (default)
  // profiling (lina_profile_enable / lina_profile_read)
  bool prof = false;
  int flags = 0;  // lina_profile_enable bits: 1 timing events, 2 skip collectives, 4 collectives only
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_gemm;  // recorded (start, end) pairs
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_a2a;   // all-to-all windows of fused passes
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_comm;  // all-to-all micro-op intervals (variable layout)
  std::vector<cudaEvent_t> prof_pool;                          // free timing events
  int64_t prof_gemm_launches = 0;
  lina::Trace* trace = nullptr;  // LINA_TRACE=1 phase trace (trace.cpp), diagnostics only
  unsigned int* route_sync = nullptr;  // zeroed words of the fused route kernel (route.cu)
  // pinned host scratch for the inference control plane (counts D2H, tables H2D)
  int* pinned = nullptr;
  size_t pinned_bytes = 0;
  // rows of the last inference call (lina_infer_last_rows): [world] each
  std::vector<int32_t> inf_recv_rows, inf_sent_rows;
  // expert packing: one NCCL communicator per packing factor m (the rank's group of m)
  std::map<int, ncclComm_t> group_comms;
  // host-bootstrap communicator (lina_comm_init_host): no NCCL; exchanges go through this
  lina_host_allgather_fn host_allgather = nullptr;
  void* host_ctx = nullptr;
};

namespace lina {
// Host allgather of `bytes` per rank through the comm's bootstrap (the caller's callback);
// throws on failure.  Only for host-bootstrap communicators.
void host_allgather(lina_comm* cm, const void* send, void* recv, size_t bytes);
// Barrier of every rank: NCCL allreduce on the dispatch communicator, or the host
// allgather of a host-bootstrap communicator (after synchronising `s`).
void comm_barrier(lina_comm* cm, cudaStream_t s);
}  // namespace lina

namespace lina {
// Profiling helpers (api.cpp): open/close one timed expert-GEMM phase on stream s.
void prof_begin(lina_comm* cm, cudaStream_t s);
void prof_end(lina_comm* cm, cudaStream_t s, int gemm_launches);
// open/close one all-to-all window of a fused pass (first mover launched .. last micro-op landed)
void prof_a2a_begin(lina_comm* cm, cudaStream_t s);
void prof_a2a_end(lina_comm* cm, cudaStream_t s);
// open/close one all-to-all micro-op (its kernels and the wait for the peers' READY)
void prof_comm_begin(lina_comm* cm, cudaStream_t s);
void prof_comm_end(lina_comm* cm, cudaStream_t s);
// Phase trace (trace.cpp): no-ops unless the comm was created with LINA_TRACE=1.
Trace* trace_create();
void trace_mark(lina_comm* cm, cudaStream_t s, const char* label);
void trace_flush(lina_comm* cm);
void trace_destroy(lina_comm* cm);
}  // namespace lina
