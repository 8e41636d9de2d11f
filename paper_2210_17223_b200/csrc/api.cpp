// C ABI of include/lina.h: argument validation (every violated invariant is
// listed), status codes, communicator lifetime, and dispatch into layer.cpp /
// infer.cpp / sched.cpp / placement.cpp.  Nothing throws across the ABI.
#include <cstring>
#include <sstream>
#include <vector>

#include "internal.h"
#include "ce.h"
#include "layer.h"
#include "kernels.h"

#include <atomic>

namespace lina {
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

static std::atomic<int64_t> g_launches{0};
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("LINA_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static cudaEvent_t prof_event(lina_comm* cm) {
  if (!cm->prof_pool.empty()) {
    cudaEvent_t e = cm->prof_pool.back();
    cm->prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  LINA_CUDA_CHECK(cudaEventCreate(&e));
  return e;
}
void prof_begin(lina_comm* cm, cudaStream_t s) {
  if (!cm->prof) return;
  cudaEvent_t a = prof_event(cm);
  LINA_CUDA_CHECK(cudaEventRecord(a, s));
  cm->prof_gemm.push_back({a, nullptr});
}
void prof_a2a_begin(lina_comm* cm, cudaStream_t s) {
  if (!cm->prof) return;
  cudaEvent_t a = prof_event(cm);
  LINA_CUDA_CHECK(cudaEventRecord(a, s));
  cm->prof_a2a.push_back({a, nullptr});
}
void prof_a2a_end(lina_comm* cm, cudaStream_t s) {
  if (!cm->prof || cm->prof_a2a.empty() || cm->prof_a2a.back().second) return;
  cudaEvent_t b = prof_event(cm);
  LINA_CUDA_CHECK(cudaEventRecord(b, s));
  cm->prof_a2a.back().second = b;
}
void prof_comm_begin(lina_comm* cm, cudaStream_t s) {
  if (!cm->prof) return;
  cudaEvent_t a = prof_event(cm);
  LINA_CUDA_CHECK(cudaEventRecord(a, s));
  cm->prof_comm.push_back({a, nullptr});
}
void prof_comm_end(lina_comm* cm, cudaStream_t s) {
  if (!cm->prof || cm->prof_comm.empty() || cm->prof_comm.back().second) return;
  cudaEvent_t b = prof_event(cm);
  LINA_CUDA_CHECK(cudaEventRecord(b, s));
  cm->prof_comm.back().second = b;
}
void prof_end(lina_comm* cm, cudaStream_t s, int gemm_launches) {
  if (!cm->prof || cm->prof_gemm.empty() || cm->prof_gemm.back().second) return;
  cudaEvent_t b = prof_event(cm);
  LINA_CUDA_CHECK(cudaEventRecord(b, s));
  cm->prof_gemm.back().second = b;
  cm->prof_gemm_launches += gemm_launches;
}

void infer_forward(lina_comm* cm, const lina_moe_desc& desc, const void* tokens,
                   const float* gate_w, const void* w1_all, const void* w2_all, void* out,
                   const lina_placement* placement, int mpd, lina_placement* plan_out, void* ws,
                   size_t ws_bytes, cudaStream_t s, const double* estimated = nullptr,
                   int32_t* replanned = nullptr);
size_t infer_workspace_bytes(const lina_moe_desc& desc, int world, int mpd);
}  // namespace lina

using namespace lina;

namespace {

template <typename F>
lina_status guarded(F&& f) {
  try {
    g_err.clear();
    return f();
  } catch (const ArgError& e) {
    g_err = e.what;
    return LINA_ERR_INVALID_ARGUMENT;
  } catch (const StatusError& e) {
    g_err = e.what;
    return e.status;
  } catch (const CudaError& e) {
    g_err = e.what;
    return LINA_ERR_CUDA;
  } catch (const NcclError& e) {
    g_err = e.what;
    return LINA_ERR_NCCL;
  } catch (const std::exception& e) {
    g_err = std::string("internal error: ") + e.what();
    return LINA_ERR_CUDA;
  }
}

// Lists every violated invariant of a descriptor (lina.h, lina_moe_desc).
void validate_desc(const lina_moe_desc* d, int world, bool static_placement) {
  if (!d) throw ArgError{"desc is NULL"};
  std::vector<std::string> v;
  const int elt = d->dtype == LINA_BF16 ? 2 : 4;
  if (d->dtype != LINA_F32 && d->dtype != LINA_BF16) v.push_back("dtype not LINA_F32/LINA_BF16");
  if (d->num_tokens < 0) v.push_back("num_tokens < 0");
  if (d->d_model <= 0) v.push_back("d_model <= 0");
  if (d->d_ffn <= 0) v.push_back("d_ffn <= 0");
  if (d->num_experts < 1 || d->num_experts > 64) v.push_back("num_experts not in [1, 64]");
  if (d->k < 1 || d->k > 8 || d->k > d->num_experts) v.push_back("k not in [1, min(E, 8)]");
  if (d->capacity < 0) v.push_back("capacity < 0 (0 = dropless)");
  if (d->n_chunks < 1 || d->n_chunks > 32 || (d->capacity >= 1 && d->n_chunks > d->capacity))
    v.push_back("n_chunks not in [1, min(C, 32)]");
  const int pack = d->pack > 1 ? d->pack : 1;
  if (d->pack < 0 || (pack & (pack - 1)) != 0 || world % pack != 0)
    v.push_back("pack not a power of two dividing world (0/1 = no packing)");
  if (static_placement && (d->capacity == 0 || pack > 1) && d->n_chunks != 1)
    v.push_back("the variable layout (capacity 0 or pack > 1) needs n_chunks == 1");
  if (d->d_model > 0 && (d->d_model * elt) % 16 != 0) v.push_back("d_model*elt % 16 != 0");
  if (d->d_ffn > 0 && (d->d_ffn * elt) % 16 != 0) v.push_back("d_ffn*elt % 16 != 0");
  if (d->d_model > 0 && d->d_model % 16 != 0) v.push_back("d_model % 16 != 0");
  if (static_placement && d->num_experts >= 1 && d->num_experts % world != 0)
    v.push_back("num_experts % world != 0 (static placement needs E_l = E/world experts per rank)");
  if (!v.empty()) {
    std::ostringstream os;
    os << "invalid lina_moe_desc:";
    for (auto& s : v) os << " [" << s << "]";
    throw ArgError{os.str()};
  }
}

// Contents of a caller-supplied placement (the tables index device buffers, so every
// entry is checked): 1 <= r_e <= min(N, max_replicas); replica devices in [0, N), distinct
// per expert, each hosting that expert; hosted ids in [-1, E), no expert twice per device,
// and every hosted expert listed among its replicas.
void validate_placement_tables(const lina_placement& pl, int E, int N, std::vector<std::string>& v) {
  const int mr = pl.max_replicas, mpd = pl.max_per_device;
  auto hosts = [&](int dv, int e) {
    for (int i = 0; i < mpd; ++i)
      if (pl.hosted[(size_t)dv * mpd + i] == e) return true;
    return false;
  };
  for (int e = 0; e < E; ++e) {
    const int r = pl.replicas[e];
    const std::string ex = "expert " + std::to_string(e);
    if (r < 1 || r > N || r > mr) {
      v.push_back(ex + ": replicas " + std::to_string(r) + " not in [1, min(num_devices, max_replicas)]");
      continue;
    }
    for (int i = 0; i < r; ++i) {
      const int dv = pl.replica_device[(size_t)e * mr + i];
      if (dv < 0 || dv >= N) {
        v.push_back(ex + ": replica device " + std::to_string(dv) + " not in [0, num_devices)");
        continue;
      }
      for (int j = 0; j < i; ++j)
        if (pl.replica_device[(size_t)e * mr + j] == dv) v.push_back(ex + ": device " + std::to_string(dv) + " listed twice");
      if (!hosts(dv, e)) v.push_back(ex + ": replica device " + std::to_string(dv) + " does not host it");
    }
  }
  for (int dv = 0; dv < N; ++dv)
    for (int i = 0; i < mpd; ++i) {
      const int e = pl.hosted[(size_t)dv * mpd + i];
      const std::string at = "hosted[" + std::to_string(dv) + "][" + std::to_string(i) + "]";
      if (e < -1 || e >= E) {
        v.push_back(at + " = " + std::to_string(e) + " not in [-1, num_experts)");
        continue;
      }
      if (e < 0) continue;
      for (int j = 0; j < i; ++j)
        if (pl.hosted[(size_t)dv * mpd + j] == e) v.push_back(at + ": expert " + std::to_string(e) + " twice");
      bool listed = false;
      const int r = std::max(0, std::min(pl.replicas[e], mr));
      for (int q = 0; q < r; ++q) listed |= pl.replica_device[(size_t)e * mr + q] == dv;
      if (!listed) v.push_back(at + ": expert " + std::to_string(e) + " not among its replica devices");
    }
  if (v.size() > 16) {  // keep the message readable; the count says how many there were
    const size_t n = v.size();
    v.resize(16);
    v.push_back("... " + std::to_string(n - 16) + " more");
  }
}

// Dropless training across ranks runs on the fused transport only (its exchanges are peer
// stores with in-kernel flags); one GPU runs both dtypes.
// A host-bootstrap communicator has no NCCL: only the fused transport's shapes run on it.
void check_host_comm(const lina_comm* cm, const lina_moe_desc* d) {
  if (!cm->host_allgather || cm->world == 1) return;
  if (d->dtype != LINA_BF16 || d->d_model % 256 != 0 || d->d_ffn % 256 != 0)
    throw StatusError{LINA_ERR_UNSUPPORTED,
                      "a host-bootstrap communicator runs the fused transport only: bf16, d_model and d_ffn "
                      "multiples of 256"};
}

void check_dropless(const lina_comm* cm, const lina_moe_desc* d) {
  check_host_comm(cm, d);
  if ((d->capacity != 0 && d->pack <= 1) || cm->world == 1) return;
  std::vector<std::string> v;
  if (cm->transport != 2 || !cm->ce) v.push_back("LINA_TRANSPORT must be fused");
  if (d->dtype != LINA_BF16) v.push_back("dtype must be bf16");
  if (d->d_model % 256 != 0 || d->d_ffn % 256 != 0) v.push_back("d_model and d_ffn must be multiples of 256");
  if (cm->world > 8 || cm->world * d->num_experts > 512) v.push_back("world <= 8 and world*E <= 512");
  if (v.empty()) return;
  std::string m = "the variable layout (capacity 0 / pack > 1) across ranks:";
  for (auto& x : v) m += " [" + x + "]";
  throw StatusError{LINA_ERR_UNSUPPORTED, m};
}

void need(std::vector<std::string>& v, const void* p, const char* name) {
  if (!p) v.push_back(std::string(name) + " is NULL");
}
void raise_if(const std::vector<std::string>& v, const char* what) {
  if (v.empty()) return;
  std::ostringstream os;
  os << what << ":";
  for (auto& s : v) os << " [" << s << "]";
  throw ArgError{os.str()};
}

}  // namespace

extern "C" {

const char* lina_last_error(void) { return g_err.c_str(); }
const char* lina_version(void) { return "lina 0.1 sm_100a"; }

lina_status lina_get_unique_id(unsigned char host_id[128]) {
  return guarded([&] {
    if (!host_id) throw ArgError{"host_id is NULL"};
    ncclUniqueId id;
    LINA_NCCL_CHECK(ncclGetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(host_id, &id, 128);
    return LINA_OK;
  });
}

}  // extern "C"

namespace {
// The device side of a communicator (streams, events, route words); rank / world set.
lina_comm* comm_base(int world, int rank, int cuda_device) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw StatusError{LINA_ERR_UNSUPPORTED, "no CUDA device visible (there is no CPU fallback)"};
  if (cuda_device < 0 || cuda_device >= ndev) throw ArgError{"cuda_device out of range"};
  LINA_CUDA_CHECK(cudaSetDevice(cuda_device));
  cudaDeviceProp prop;
  LINA_CUDA_CHECK(cudaGetDeviceProperties(&prop, cuda_device));
  if (prop.major != 10)
    throw StatusError{LINA_ERR_UNSUPPORTED, "device is sm_" + std::to_string(prop.major) +
                                                std::to_string(prop.minor) + "; this library is built for sm_100a only"};
  auto* cm = new lina_comm();
  cm->rank = rank;
  cm->world = world;
  cm->device = cuda_device;
  cm->num_sms = prop.multiProcessorCount;
  int lo_prio = 0, hi_prio = 0;
  LINA_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
  LINA_CUDA_CHECK(cudaStreamCreateWithPriority(&cm->hi, cudaStreamNonBlocking, hi_prio));
  LINA_CUDA_CHECK(cudaStreamCreateWithPriority(&cm->hi2, cudaStreamNonBlocking, hi_prio));
  LINA_CUDA_CHECK(cudaStreamCreateWithPriority(&cm->lo, cudaStreamNonBlocking, lo_prio));
  LINA_CUDA_CHECK(cudaMalloc(&cm->route_sync, sizeof(unsigned int) * route_sync_words()));
  LINA_CUDA_CHECK(cudaMemset(cm->route_sync, 0, sizeof(unsigned int) * route_sync_words()));
  {  // dynamic tile schedule of the expert GEMMs (gemm_tc.cu): LINA_GEMM_DYN=0 keeps the static one
    const char* dv = getenv("LINA_GEMM_DYN");
    if (!(dv && dv[0] == '0')) {
      LINA_CUDA_CHECK(cudaMalloc(&cm->tile_ctr, sizeof(unsigned int)));
      LINA_CUDA_CHECK(cudaMemset(cm->tile_ctr, 0, sizeof(unsigned int)));
    }
  }
  cm->ev.resize(128);
  for (auto& e : cm->ev) LINA_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const char* trv = getenv("LINA_TRACE");
  if (trv && atoi(trv) > 0) cm->trace = trace_create();
  return cm;
}
}  // namespace

namespace lina {
void host_allgather(lina_comm* cm, const void* send, void* recv, size_t bytes) {
  if (!cm->host_allgather) throw StatusError{LINA_ERR_UNSUPPORTED, "host allgather on an NCCL communicator"};
  if (cm->host_allgather(send, recv, bytes, cm->host_ctx) != 0)
    throw StatusError{LINA_ERR_CUDA, "host allgather callback failed"};
}
void comm_barrier(lina_comm* cm, cudaStream_t s) {
  if (cm->world == 1) {
    LINA_CUDA_CHECK(cudaStreamSynchronize(s));
    return;
  }
  if (cm->host_allgather) {
    LINA_CUDA_CHECK(cudaStreamSynchronize(s));
    std::vector<int> all((size_t)cm->world);
    const int one = 1;
    host_allgather(cm, &one, all.data(), sizeof(int));
    return;
  }
  int* one = nullptr;
  LINA_CUDA_CHECK(cudaMallocAsync((void**)&one, sizeof(int), s));
  LINA_CUDA_CHECK(cudaMemsetAsync(one, 0, sizeof(int), s));
  LINA_NCCL_CHECK(ncclAllReduce(one, one, 1, ncclInt32, ncclSum, cm->ep_disp, s));
  LINA_CUDA_CHECK(cudaFreeAsync(one, s));
  LINA_CUDA_CHECK(cudaStreamSynchronize(s));
}
}  // namespace lina

extern "C" {

lina_status lina_comm_init(int world, int rank, int cuda_device, const unsigned char* host_id,
                           int nccl_max_ctas, lina_comm** out) {
  return guarded([&] {
    std::vector<std::string> v;
    if (!out) v.push_back("out is NULL");
    if (world < 1) v.push_back("world < 1");
    if (rank < 0 || rank >= world) v.push_back("rank not in [0, world)");
    if (world > 1 && !host_id) v.push_back("host_id is NULL with world > 1");
    if (nccl_max_ctas < 0) v.push_back("nccl_max_ctas < 0");
    raise_if(v, "lina_comm_init");
    lina_comm* cm = comm_base(world, rank, cuda_device);
    if (world > 1) {
      ncclUniqueId id;
      std::memcpy(&id, host_id, 128);
      ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
      if (nccl_max_ctas > 0) cfg.maxCTAs = nccl_max_ctas;
      LINA_NCCL_CHECK(ncclCommInitRankConfig(&cm->ep_disp, world, id, rank, &cfg));
      ncclConfig_t cfg2 = NCCL_CONFIG_INITIALIZER;
      if (nccl_max_ctas > 0) cfg2.maxCTAs = nccl_max_ctas;
      LINA_NCCL_CHECK(ncclCommSplit(cm->ep_disp, 0, rank, &cm->ep_comb, &cfg2));
      // DP communicator (allreduce micro-ops): its CTA budget is separate from the EP
      // ones — under the LINA policy its micro-ops run in the windows without all-to-all
      // traffic, so it keeps NCCL's default CTA count (LINA_DP_MAX_CTAS overrides).
      ncclConfig_t cfg3 = NCCL_CONFIG_INITIALIZER;
      const char* dpc = getenv("LINA_DP_MAX_CTAS");
      const int dp_ctas = dpc ? atoi(dpc) : 0;
      if (dp_ctas > 0) cfg3.maxCTAs = dp_ctas;
      LINA_NCCL_CHECK(ncclCommSplit(cm->ep_disp, 0, rank, &cm->dp, &cfg3));
      cm->sched = sched_create(cm);
      // Training all-to-all transport (LINA_TRANSPORT): "fused" (default) = peer stores from
      // the permute / combine-backward kernels and the GEMM epilogues; "ce" = copy engines
      // over NVLink (zero SMs, ce.cpp); "nccl" = ncclAlltoAll micro-ops, whose kernels run
      // beside the persistent expert GEMM and need SMs left free for them.
      const char* tr = getenv("LINA_TRANSPORT");
      const std::string t = tr ? tr : "fused";
      cm->transport = t == "nccl" ? 0 : (t == "ce" ? 1 : 2);
      if (cm->transport > 0) cm->ce = new CeTransport(cm);
      tc_set_reserved_sms(cm->ce ? 0 : (nccl_max_ctas > 0 ? 2 * nccl_max_ctas : 16));
    }
    *out = cm;
    return LINA_OK;
  });
}

lina_status lina_comm_init_host(int world, int rank, int cuda_device, lina_host_allgather_fn fn, void* ctx,
                                lina_comm** out) {
  return guarded([&] {
    std::vector<std::string> v;
    if (!out) v.push_back("out is NULL");
    if (world < 1) v.push_back("world < 1");
    if (rank < 0 || rank >= world) v.push_back("rank not in [0, world)");
    if (!fn) v.push_back("fn is NULL");
    raise_if(v, "lina_comm_init_host");
    lina_comm* cm = comm_base(world, rank, cuda_device);
    cm->host_allgather = fn;
    cm->host_ctx = ctx;
    if (world > 1) {
      cm->transport = 2;  // fused: its exchanges are peer stores, its bootstrap host-side
      cm->ce = new CeTransport(cm);
      tc_set_reserved_sms(0);
    }
    *out = cm;
    return LINA_OK;
  });
}

lina_status lina_comm_destroy(lina_comm* cm) {
  return guarded([&] {
    if (!cm) return LINA_OK;
    cudaSetDevice(cm->device);
    trace_destroy(cm);
    if (cm->sched) sched_destroy(cm->sched);
    cm->sched = nullptr;
    delete cm->ce;
    cm->ce = nullptr;
    for (auto& kv : cm->group_comms) ncclCommDestroy(kv.second);
    cm->group_comms.clear();
    if (cm->dp) ncclCommDestroy(cm->dp);
    if (cm->ep_comb) ncclCommDestroy(cm->ep_comb);
    if (cm->ep_disp) ncclCommDestroy(cm->ep_disp);
    for (auto e : cm->ev) cudaEventDestroy(e);
    if (cm->hi) cudaStreamDestroy(cm->hi);
    if (cm->hi2) cudaStreamDestroy(cm->hi2);
    if (cm->lo) cudaStreamDestroy(cm->lo);
    for (auto e : cm->prof_pool) cudaEventDestroy(e);
    if (cm->pinned) cudaFreeHost(cm->pinned);
    if (cm->route_sync) cudaFree(cm->route_sync);
    if (cm->tile_ctr) {
      tc_set_tile_counter(nullptr);
      cudaFree(cm->tile_ctr);
    }
    delete cm;
    return LINA_OK;
  });
}

lina_status lina_comm_check(lina_comm* cm) {
  return guarded([&] {
    if (!cm) throw ArgError{"comm is NULL"};
    LINA_CUDA_CHECK(cudaPeekAtLastError());
    if (cm->sched) sched_check(cm->sched);
    for (ncclComm_t c : {cm->ep_disp, cm->ep_comb, cm->dp}) {
      if (!c) continue;
      ncclResult_t r = ncclSuccess;
      LINA_NCCL_CHECK(ncclCommGetAsyncError(c, &r));
      if (r != ncclSuccess && r != ncclInProgress)
        throw NcclError{std::string("async NCCL error: ") + ncclGetErrorString(r)};
    }
    return LINA_OK;
  });
}

lina_status lina_comm_info(const lina_comm* cm, int* rank, int* world) {
  return guarded([&] {
    if (!cm) throw ArgError{"comm is NULL"};
    if (rank) *rank = cm->rank;
    if (world) *world = cm->world;
    return LINA_OK;
  });
}

lina_status lina_placement_compute(const double* pop, int32_t E, int32_t N, int32_t mpd,
                                   lina_placement* out) {
  return guarded([&] {
    std::vector<std::string> v;
    need(v, pop, "host_popularity");
    need(v, out, "out");
    if (E < 1) v.push_back("num_experts < 1");
    if (N < 1) v.push_back("num_devices < 1");
    if (mpd < 1) v.push_back("max_per_device < 1");
    if (out) {
      need(v, out->replicas, "out->replicas");
      need(v, out->replica_device, "out->replica_device");
      need(v, out->hosted, "out->hosted");
      if (out->max_replicas < std::min(N, 1 << 30) && out->max_replicas < N)
        v.push_back("out->max_replicas < num_devices");
    }
    if (pop)
      for (int e = 0; e < E; ++e)
        if (!(pop[e] >= 0.0)) {
          v.push_back("popularity[" + std::to_string(e) + "] < 0 or NaN");
          break;
        }
    raise_if(v, "lina_placement_compute");
    std::string err;
    lina_status st = placement_compute(pop, E, N, mpd, out, &err);
    if (st != LINA_OK) throw StatusError{st, err};
    return LINA_OK;
  });
}

lina_status lina_replica_split(int32_t count, int32_t replicas, int32_t source_rank,
                               int32_t* host_out) {
  return guarded([&] {
    std::vector<std::string> v;
    if (count < 0) v.push_back("count < 0");
    if (replicas < 1) v.push_back("replicas < 1");
    if (source_rank < 0) v.push_back("source_rank < 0");
    need(v, host_out, "host_out");
    raise_if(v, "lina_replica_split");
    replica_split(count, replicas, source_rank, host_out);
    return LINA_OK;
  });
}

lina_status lina_popprof_create(int32_t L, int32_t E, int32_t k, int32_t l, lina_pop_profile** out) {
  return guarded([&] {
    std::vector<std::string> v;
    need(v, out, "out");
    if (L < 2) v.push_back("num_layers < 2");
    if (E < 1) v.push_back("num_experts < 1");
    if (k < 1 || k > E) v.push_back("k outside [1, num_experts]");
    if (l < 1 || l >= L) v.push_back("path_len outside [1, num_layers)");
    raise_if(v, "lina_popprof_create");
    *out = popprof_create(L, E, k, l);
    return LINA_OK;
  });
}

lina_status lina_popprof_destroy(lina_pop_profile* prof) {
  delete prof;
  return LINA_OK;
}

lina_status lina_popprof_add(lina_pop_profile* prof, const int32_t* sel, int64_t T) {
  return guarded([&] {
    std::vector<std::string> v;
    need(v, prof, "prof");
    if (T < 0) v.push_back("num_tokens < 0");
    if (T > 0) need(v, sel, "host_sel");
    if (prof && sel && T > 0) {
      const std::string bad = popprof_check_ids(prof, sel, T, prof->L);
      if (!bad.empty()) v.push_back(bad);
    }
    raise_if(v, "lina_popprof_add");
    popprof_add(prof, sel, T);
    return LINA_OK;
  });
}

lina_status lina_popprof_estimate(const lina_pop_profile* prof, int32_t layer, const int32_t* hist,
                                  int64_t T, double* pop, int32_t* topk) {
  return guarded([&] {
    std::vector<std::string> v;
    need(v, prof, "prof");
    need(v, pop, "host_popularity");
    if (T < 0) v.push_back("num_tokens < 0");
    if (T > 0) need(v, hist, "host_history");
    if (prof) {
      if (layer < prof->l) v.push_back("layer < path_len (no sample path yet)");
      if (layer >= prof->L) v.push_back("layer >= num_layers");
      if (hist && T > 0) {
        const std::string bad = popprof_check_ids(prof, hist, T, prof->l);
        if (!bad.empty()) v.push_back(bad);
      }
    }
    raise_if(v, "lina_popprof_estimate");
    popprof_estimate(prof, layer, hist, T, pop, topk);
    return LINA_OK;
  });
}

lina_status lina_popprof_save(const lina_pop_profile* prof, const char* path) {
  return guarded([&] {
    std::vector<std::string> v;
    need(v, prof, "prof");
    need(v, path, "path");
    raise_if(v, "lina_popprof_save");
    const std::string err = popprof_save(prof, path);
    if (!err.empty()) throw ArgError{"lina_popprof_save: " + err};
    return LINA_OK;
  });
}

lina_status lina_popprof_info(const lina_pop_profile* prof, int32_t* L, int32_t* E, int32_t* k, int32_t* l) {
  if (!prof) {
    set_error("lina_popprof_info: prof is NULL");
    return LINA_ERR_INVALID_ARGUMENT;
  }
  if (L) *L = prof->L;
  if (E) *E = prof->E;
  if (k) *k = prof->k;
  if (l) *l = prof->l;
  return LINA_OK;
}

lina_status lina_popprof_load(const char* path, lina_pop_profile** out) {
  return guarded([&] {
    std::vector<std::string> v;
    need(v, path, "path");
    need(v, out, "out");
    raise_if(v, "lina_popprof_load");
    const std::string err = popprof_load(path, out);
    if (!err.empty()) throw ArgError{"lina_popprof_load: " + err};
    return LINA_OK;
  });
}

lina_status lina_phase_two_check(const double* est, const int32_t* actual, int32_t E, int32_t k,
                                 int32_t* identical) {
  return guarded([&] {
    std::vector<std::string> v;
    need(v, est, "host_estimated");
    need(v, actual, "host_actual_counts");
    need(v, identical, "host_identical");
    if (E < 1) v.push_back("num_experts < 1");
    if (k < 1) v.push_back("k < 1");
    raise_if(v, "lina_phase_two_check");
    *identical = phase_two_identical(est, actual, E, k) ? 1 : 0;
    return LINA_OK;
  });
}

lina_status lina_moe_workspace_size(const lina_comm* cm, const lina_moe_desc* desc,
                                    size_t* workspace_bytes, size_t* saved_bytes) {
  return guarded([&] {
    if (!cm) throw ArgError{"comm is NULL"};
    validate_desc(desc, cm->world, true);
    check_dropless(cm, desc);
    Plan p = make_plan(*desc, cm->world);
    if (workspace_bytes) *workspace_bytes = p.ws_bytes;
    if (saved_bytes) *saved_bytes = p.saved_bytes;
    return LINA_OK;
  });
}

lina_status lina_moe_forward(lina_comm* cm, const lina_moe_desc* desc, const void* tokens,
                             const float* gate_w, const void* w1, const void* w2, void* out,
                             void* saved, void* workspace, size_t workspace_bytes,
                             lina_route* route, lina_stream stream) {
  return guarded([&] {
    if (!cm) throw ArgError{"comm is NULL"};
    validate_desc(desc, cm->world, true);
    check_dropless(cm, desc);
    std::vector<std::string> v;
    const bool any = desc->num_tokens > 0;
    if (any) need(v, tokens, "tokens");
    need(v, gate_w, "gate_w");
    need(v, w1, "w1");
    need(v, w2, "w2");
    if (any) need(v, out, "out");
    need(v, saved, "saved (forward keeps routing and expert activations there)");
    need(v, workspace, "workspace");
    if (route && route->override_routing) {
      need(v, route->idx, "route->idx (override_routing)");
      need(v, route->gate, "route->gate (override_routing)");
    }
    raise_if(v, "lina_moe_forward");
    Plan p = make_plan(*desc, cm->world);
    if (workspace_bytes < p.ws_bytes)
      throw StatusError{LINA_ERR_WORKSPACE, "workspace_bytes " + std::to_string(workspace_bytes) +
                                                " < required " + std::to_string(p.ws_bytes)};
    LINA_CUDA_CHECK(cudaSetDevice(cm->device));
    tc_set_tile_counter(cm->tile_ctr);
    moe_forward(cm, p, tokens, gate_w, w1, w2, out, saved, workspace, route, (cudaStream_t)stream);
    return LINA_OK;
  });
}

lina_status lina_moe_backward(lina_comm* cm, const lina_moe_desc* desc, const void* saved,
                              const void* dout, const void* tokens, const float* gate_w,
                              const void* w1, const void* w2, void* dtokens, float* dgate_w,
                              void* dw1, void* dw2, void* workspace, size_t workspace_bytes,
                              lina_stream stream) {
  return guarded([&] {
    if (!cm) throw ArgError{"comm is NULL"};
    validate_desc(desc, cm->world, true);
    check_dropless(cm, desc);
    std::vector<std::string> v;
    const bool any = desc->num_tokens > 0;
    need(v, saved, "saved");
    if (any) {
      need(v, dout, "dout");
      need(v, tokens, "tokens");
      need(v, dtokens, "dtokens");
    }
    need(v, gate_w, "gate_w");
    need(v, w1, "w1");
    need(v, w2, "w2");
    need(v, dgate_w, "dgate_w");
    need(v, dw1, "dw1");
    need(v, dw2, "dw2");
    need(v, workspace, "workspace");
    raise_if(v, "lina_moe_backward");
    Plan p = make_plan(*desc, cm->world);
    if (workspace_bytes < p.ws_bytes)
      throw StatusError{LINA_ERR_WORKSPACE, "workspace_bytes " + std::to_string(workspace_bytes) +
                                                " < required " + std::to_string(p.ws_bytes)};
    LINA_CUDA_CHECK(cudaSetDevice(cm->device));
    tc_set_tile_counter(cm->tile_ctr);
    moe_backward(cm, p, saved, dout, tokens, gate_w, w1, w2, dtokens, dgate_w, dw1, dw2, workspace,
                 (cudaStream_t)stream);
    return LINA_OK;
  });
}

lina_status lina_moe_infer_workspace_size(const lina_comm* cm, const lina_moe_desc* desc,
                                          int32_t max_per_device, size_t* workspace_bytes) {
  return guarded([&] {
    if (!cm) throw ArgError{"comm is NULL"};
    validate_desc(desc, cm->world, false);
    if (max_per_device < 1) throw ArgError{"max_per_device < 1"};
    if (workspace_bytes) *workspace_bytes = infer_workspace_bytes(*desc, cm->world, max_per_device);
    return LINA_OK;
  });
}

// Validation and dispatch shared by lina_moe_infer_forward and its two-phase variant
// (estimated != NULL: phase-two check against the phase-one `placement`).
static lina_status infer_entry(lina_comm* cm, const lina_moe_desc* desc, const void* tokens,
                               const float* gate_w, const void* w1_all, const void* w2_all, void* out,
                               const lina_placement* placement, int32_t max_per_device,
                               lina_placement* plan_out, void* workspace, size_t workspace_bytes,
                               lina_stream stream, const double* estimated, int32_t* replanned,
                               const char* what) {
  return guarded([&] {
    if (!cm) throw ArgError{"comm is NULL"};
    validate_desc(desc, cm->world, false);
    std::vector<std::string> v;
    if (desc->num_tokens > 0) {
      need(v, tokens, "tokens");
      need(v, out, "out");
    }
    need(v, gate_w, "gate_w");
    need(v, w1_all, "w1_all");
    need(v, w2_all, "w2_all");
    need(v, workspace, "workspace");
    if (!placement && max_per_device < 1) v.push_back("max_per_device < 1 with placement == NULL");
    if (placement) {
      if (placement->num_experts != desc->num_experts) v.push_back("placement->num_experts != E");
      if (placement->num_devices != cm->world) v.push_back("placement->num_devices != world");
      if (placement->max_per_device < 1) v.push_back("placement->max_per_device < 1");
      if (placement->max_replicas < 1) v.push_back("placement->max_replicas < 1");
      need(v, placement->replicas, "placement->replicas");
      need(v, placement->replica_device, "placement->replica_device");
      need(v, placement->hosted, "placement->hosted");
      if (v.empty()) validate_placement_tables(*placement, desc->num_experts, cm->world, v);
    }
    if (plan_out) {
      need(v, plan_out->replicas, "plan_out->replicas");
      need(v, plan_out->replica_device, "plan_out->replica_device");
      need(v, plan_out->hosted, "plan_out->hosted");
      if (plan_out->max_replicas < cm->world) v.push_back("plan_out->max_replicas < world");
    }
    raise_if(v, what);
    const int mpd = placement ? placement->max_per_device : max_per_device;
    if (workspace_bytes < infer_workspace_bytes(*desc, cm->world, mpd))
      throw StatusError{LINA_ERR_WORKSPACE, "workspace_bytes < lina_moe_infer_workspace_size"};
    LINA_CUDA_CHECK(cudaSetDevice(cm->device));
    tc_set_tile_counter(cm->tile_ctr);
    infer_forward(cm, *desc, tokens, gate_w, w1_all, w2_all, out, placement, max_per_device,
                  plan_out, workspace, workspace_bytes, (cudaStream_t)stream, estimated, replanned);
    return LINA_OK;
  });
}

lina_status lina_moe_infer_forward(lina_comm* cm, const lina_moe_desc* desc, const void* tokens,
                                   const float* gate_w, const void* w1_all, const void* w2_all,
                                   void* out, const lina_placement* placement,
                                   int32_t max_per_device, lina_placement* plan_out,
                                   void* workspace, size_t workspace_bytes, lina_stream stream) {
  return infer_entry(cm, desc, tokens, gate_w, w1_all, w2_all, out, placement, max_per_device, plan_out,
                     workspace, workspace_bytes, stream, nullptr, nullptr, "lina_moe_infer_forward");
}

lina_status lina_moe_infer_forward_two_phase(lina_comm* cm, const lina_moe_desc* desc,
                                             const void* tokens, const float* gate_w,
                                             const void* w1_all, const void* w2_all, void* out,
                                             const lina_placement* placement,
                                             const double* estimated, lina_placement* plan_out,
                                             int32_t* replanned, void* workspace,
                                             size_t workspace_bytes, lina_stream stream) {
  if (!placement || !estimated) {
    set_error(std::string("lina_moe_infer_forward_two_phase:") +
              (placement ? "" : " placement (the phase-one plan) is NULL;") +
              (estimated ? "" : " host_estimated is NULL;"));
    return LINA_ERR_INVALID_ARGUMENT;
  }
  if (desc)
    for (int e = 0; e < desc->num_experts; ++e)
      if (!(estimated[e] >= 0.0)) {
        set_error("lina_moe_infer_forward_two_phase: host_estimated[" + std::to_string(e) + "] < 0 or NaN");
        return LINA_ERR_INVALID_ARGUMENT;
      }
  return infer_entry(cm, desc, tokens, gate_w, w1_all, w2_all, out, placement, placement->max_per_device,
                     plan_out, workspace, workspace_bytes, stream, estimated, replanned,
                     "lina_moe_infer_forward_two_phase");
}

lina_status lina_pack_weights(lina_comm* cm, int32_t num_experts, int32_t pack_from, int32_t pack_to,
                              size_t expert_elems, lina_dtype dtype, const void* w_from, void* w_to,
                              lina_stream stream) {
  return guarded([&] {
    std::vector<std::string> v;
    if (!cm) throw ArgError{"comm is NULL"};
    const int P = cm->world;
    auto pow2_div = [&](int m) { return m >= 1 && (m & (m - 1)) == 0 && P % m == 0; };
    if (num_experts < 1 || num_experts % P != 0) v.push_back("num_experts not a positive multiple of world");
    if (!pow2_div(pack_from)) v.push_back("pack_from not a power of two dividing world");
    if (!pow2_div(pack_to)) v.push_back("pack_to not a power of two dividing world");
    if (dtype != LINA_F32 && dtype != LINA_BF16) v.push_back("dtype not LINA_F32/LINA_BF16");
    if (expert_elems == 0) v.push_back("expert_elems == 0");
    need(v, w_from, "w_from");
    need(v, w_to, "w_to");
    if (P > 1 && !cm->ce) v.push_back("world > 1 needs the fused or ce transport (peer mappings)");
    raise_if(v, "lina_pack_weights");
    LINA_CUDA_CHECK(cudaSetDevice(cm->device));
    tc_set_tile_counter(cm->tile_ctr);
    pack_weights(cm, num_experts, pack_from, pack_to, expert_elems * (dtype == LINA_BF16 ? 2 : 4), w_from, w_to,
                 (cudaStream_t)stream);
    return LINA_OK;
  });
}

lina_status lina_infer_last_rows(const lina_comm* cm, int32_t* recv_rows, int32_t* sent_rows) {
  return guarded([&] {
    if (!cm) throw ArgError{"comm is NULL"};
    for (int r = 0; r < cm->world; ++r) {
      if (recv_rows) recv_rows[r] = r < (int)cm->inf_recv_rows.size() ? cm->inf_recv_rows[r] : 0;
      if (sent_rows) sent_rows[r] = r < (int)cm->inf_sent_rows.size() ? cm->inf_sent_rows[r] : 0;
    }
    return LINA_OK;
  });
}

lina_status lina_sched_config(lina_comm* cm, lina_policy policy, size_t partition_bytes) {
  return guarded([&] {
    if (!cm) throw ArgError{"comm is NULL"};
    if (policy != LINA_SCHED_BASELINE && policy != LINA_SCHED_LINA && policy != LINA_SCHED_NAIVE &&
        policy != LINA_SCHED_DEFER)
      throw ArgError{"policy not LINA_SCHED_BASELINE/LINA/NAIVE/DEFER"};
    if (cm->sched) sched_config(cm->sched, policy, partition_bytes);
    return LINA_OK;
  });
}

lina_status lina_allreduce_submit(lina_comm* cm, void* grad, size_t count, lina_dtype dtype,
                                  lina_stream ready_stream) {
  return guarded([&] {
    std::vector<std::string> v;
    if (!cm) v.push_back("comm is NULL");
    need(v, grad, "grad");
    if (dtype != LINA_F32 && dtype != LINA_BF16) v.push_back("dtype not LINA_F32/LINA_BF16");
    raise_if(v, "lina_allreduce_submit");
    if (!cm->sched && cm->world > 1)
      throw StatusError{LINA_ERR_UNSUPPORTED, "allreduce needs an NCCL communicator (lina_comm_init)"};
    if (count == 0 || !cm->sched) return LINA_OK;  // world == 1: the sum over one rank is itself
    LINA_CUDA_CHECK(cudaSetDevice(cm->device));
    tc_set_tile_counter(cm->tile_ctr);
    sched_submit(cm->sched, grad, count, dtype, (cudaStream_t)ready_stream);
    return LINA_OK;
  });
}

lina_status lina_allreduce_wait(lina_comm* cm, lina_stream stream) {
  return guarded([&] {
    if (!cm) throw ArgError{"comm is NULL"};
    if (cm->sched) sched_wait(cm->sched, (cudaStream_t)stream);
    return LINA_OK;
  });
}

lina_status lina_profile_enable(lina_comm* cm, int on) {
  return guarded([&] {
    if (!cm) throw ArgError{"comm is NULL"};
    if (on < 0 || on > 7 || ((on & 2) && (on & 4)))
      throw ArgError{"profile flags: 1 timing | 2 skip collectives | 4 collectives only (2 and 4 exclusive)"};
    cm->prof = (on & 1) != 0;
    cm->flags = on;
    return LINA_OK;
  });
}

lina_status lina_profile_read(lina_comm* cm, lina_profile* out) {
  return guarded([&] {
    if (!cm) throw ArgError{"comm is NULL"};
    if (!out) throw ArgError{"out is NULL"};
    double ms = 0.0;
    int64_t phases = 0;
    // timestamps relative to one reference event (all events are on this device)
    cudaEvent_t ref = !cm->prof_gemm.empty()  ? cm->prof_gemm.front().first
                      : !cm->prof_a2a.empty() ? cm->prof_a2a.front().first
                      : !cm->prof_comm.empty() ? cm->prof_comm.front().first
                                               : nullptr;
    auto at = [&](cudaEvent_t e) {
      float t = 0.f;
      LINA_CUDA_CHECK(cudaEventSynchronize(e));
      LINA_CUDA_CHECK(cudaEventElapsedTime(&t, ref, e));
      return (double)t;
    };
    std::vector<std::pair<double, double>> gemm_iv;
    for (auto& pr : cm->prof_gemm) {
      if (pr.second) {
        const double a = at(pr.first), b = at(pr.second);
        ms += b - a;
        gemm_iv.push_back({a, b});
        ++phases;
      }
    }
    // all-to-all windows of the fused passes and the expert-GEMM time inside them (the
    // paper's pipelining efficiency: non-idle time of the computation stream
    // during the all-to-all)
    double win = 0.0, busy = 0.0;
    int64_t nwin = 0;
    for (auto& pr : cm->prof_a2a) {
      if (!pr.second) continue;
      const double a = at(pr.first), b = at(pr.second);
      win += b - a;
      ++nwin;
      for (auto& g : gemm_iv) busy += std::max(0.0, std::min(b, g.second) - std::max(a, g.first));
    }
    double comm = 0.0;
    int64_t ncomm = 0;
    for (auto& pr : cm->prof_comm) {
      if (!pr.second) continue;
      comm += at(pr.second) - at(pr.first);
      ++ncomm;
    }
    for (auto* v : {&cm->prof_gemm, &cm->prof_a2a, &cm->prof_comm}) {
      for (auto& pr : *v) {
        if (pr.second) cm->prof_pool.push_back(pr.second);
        cm->prof_pool.push_back(pr.first);
      }
      v->clear();
    }
    out->kernel_launches = g_launches.exchange(0);
    out->gemm_launches = cm->prof_gemm_launches;
    out->gemm_ms = ms;
    out->gemm_phases = phases;
    out->a2a_window_ms = win;
    out->gemm_in_a2a_ms = busy;
    out->a2a_windows = nwin;
    out->a2a_op_ms = comm;
    out->a2a_ops = ncomm;
    cm->prof_gemm_launches = 0;
    return LINA_OK;
  });
}

lina_status lina_sched_stats(lina_comm* cm, int64_t* issued, int64_t* deferred) {
  return guarded([&] {
    if (!cm) throw ArgError{"comm is NULL"};
    int64_t a = 0, b = 0;
    if (cm->sched) sched_stats(cm->sched, &a, &b);
    if (issued) *issued = a;
    if (deferred) *deferred = b;
    return LINA_OK;
  });
}

}  // extern "C"
