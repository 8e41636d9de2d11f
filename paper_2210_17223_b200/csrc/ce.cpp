// Copy-engine all-to-all transport over NVLink 5 / NVSwitch (zero SMs).
//
// The all-to-all micro-ops of the training layer move fixed,
// host-known block sizes, so they need no kernel at all: every rank maps its peers'
// send buffers (CUDA IPC) and PULLS the blocks addressed to it with one
// cudaMemcpyAsync per (peer, chunk) on a per-peer high-priority stream — the copy
// engines move the bytes and every SM stays with the expert GEMM (an NCCL all-to-all
// at NVLink rate occupies ~16 CTAs per communicator, measured).
// Ordering across ranks uses stream memory operations on a small flag array that
// every rank maps from every peer:
//   READY[x][src][c]  (at the receiver) = seq  : src's block of exchange x, chunk c is written
//   PULLED[x][dst]    (at the sender)   = seq  : dst has copied everything it needs of x
// The producer writes READY into every peer after its kernel (cuStreamWriteValue32,
// ordered after the kernel, with the default memory barrier); the consumer's pull
// stream waits for it (cuStreamWaitValue32 >= seq) and writes PULLED back after its
// copies; a producer waits for PULLED of the previous round before it overwrites its
// send buffer.  seq counts forward (backward) passes on every rank identically.
// No rank ever spins in a kernel on another rank's memory.
#include <cuda.h>

#include <cstring>
#include <map>

#include "ce.h"

namespace lina {

typedef CUresult (*WaitValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*WriteValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
typedef CUresult (*PtrAttrFn)(void*, CUpointer_attribute, CUdeviceptr);

static void* entry(const char* name) {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return f;
}

struct CeTransport::Impl {
  WaitValueFn wait_fn = nullptr;
  WriteValueFn write_fn = nullptr;
  AddrRangeFn range_fn = nullptr;
  PtrAttrFn attr_fn = nullptr;
  // IPC-opened peer allocation bases, keyed by (rank, handle bytes)
  std::map<std::pair<int, std::string>, char*> opened;
  // mapped peer pointers for a local pointer, with the allocation's buffer id and the
  // mapping generation
  struct Mapping {
    unsigned long long buffer_id = 0;
    uint64_t gen = 0;
    std::vector<char*> ptrs;
  };
  std::map<const void*, Mapping> maps;
  uint64_t next_gen = 0;
  // device copies of peer pointer arrays (with the generation they were built from)
  std::map<std::pair<const void*, size_t>, std::pair<void*, uint64_t>> ptr_arrays;
  unsigned long long buffer_id(const void* p) const {
    unsigned long long id = 0;
    if (attr_fn(&id, CU_POINTER_ATTRIBUTE_BUFFER_ID, (CUdeviceptr)p) != CUDA_SUCCESS)
      throw CudaError{"cuPointerGetAttribute(BUFFER_ID) failed: not a device allocation"};
    return id;
  }
  void* stage = nullptr;  // device staging for handle exchange
};

void* const* CeTransport::dev_ptrs(const void* local, size_t offset, cudaStream_t s, uint64_t layout_key) {
  const auto& pr = peers(local, s, layout_key);  // (re-)maps first if the allocation changed
  const uint64_t gen = generation(local);
  auto key = std::make_pair(local, offset);
  auto it = impl_->ptr_arrays.find(key);
  if (it != impl_->ptr_arrays.end()) {
    if (it->second.second == gen) return (void* const*)it->second.first;
    LINA_CUDA_CHECK(cudaFree(it->second.first));  // built from a stale mapping
    impl_->ptr_arrays.erase(it);
  }
  std::vector<char*> v(pr.size());
  for (size_t i = 0; i < pr.size(); ++i) v[i] = pr[i] + offset;
  void* d = nullptr;
  LINA_CUDA_CHECK(cudaMalloc(&d, sizeof(char*) * v.size()));
  LINA_CUDA_CHECK(cudaMemcpy(d, v.data(), sizeof(char*) * v.size(), cudaMemcpyHostToDevice));
  impl_->ptr_arrays[key] = {d, gen};
  return (void* const*)d;
}

CeTransport::CeTransport(lina_comm* cm) : cm_(cm), impl_(new Impl) {
  impl_->wait_fn = (WaitValueFn)entry("cuStreamWaitValue32");
  impl_->write_fn = (WriteValueFn)entry("cuStreamWriteValue32");
  impl_->range_fn = (AddrRangeFn)entry("cuMemGetAddressRange");
  impl_->attr_fn = (PtrAttrFn)entry("cuPointerGetAttribute");
  if (!impl_->wait_fn || !impl_->write_fn || !impl_->range_fn || !impl_->attr_fn)
    throw StatusError{LINA_ERR_UNSUPPORTED, "stream memory operations not available"};
  const int P = cm->world;
  nflags_ = (size_t)kKinds * P * kMaxChunks;
  LINA_CUDA_CHECK(cudaMalloc(&flags_, nflags_ * sizeof(uint32_t)));
  LINA_CUDA_CHECK(cudaMemset(flags_, 0, nflags_ * sizeof(uint32_t)));
  LINA_CUDA_CHECK(cudaMalloc(&impl_->stage, 128 * (size_t)P));
  LINA_CUDA_CHECK(cudaMalloc(&done_, kDoneSites * sizeof(unsigned int)));
  LINA_CUDA_CHECK(cudaMemset(done_, 0, kDoneSites * sizeof(unsigned int)));
  LINA_CUDA_CHECK(cudaMalloc(&rounds_, 3 * sizeof(uint32_t)));
  LINA_CUDA_CHECK(cudaMemset(rounds_, 0, 3 * sizeof(uint32_t)));
  peer_slots_.assign(kKinds, nullptr);
  peer_flags_ = map_collective(flags_, cm->hi, 0);
  for (int r = 0; r < P; ++r) {
    cudaStream_t a, b;
    int lo_prio = 0, hi_prio = 0;
    LINA_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    LINA_CUDA_CHECK(cudaStreamCreateWithPriority(&a, cudaStreamNonBlocking, hi_prio));
    LINA_CUDA_CHECK(cudaStreamCreateWithPriority(&b, cudaStreamNonBlocking, hi_prio));
    disp_.push_back(a);
    comb_.push_back(b);
  }
  events_.resize((size_t)4 * P * (kMaxChunks + 2));
  for (auto& e : events_) LINA_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

CeTransport::~CeTransport() {
  cudaDeviceSynchronize();
  for (auto& kv : impl_->opened) cudaIpcCloseMemHandle(kv.second);
  for (auto& kv : impl_->ptr_arrays) cudaFree(kv.second.first);
  for (auto s : disp_) cudaStreamDestroy(s);
  for (auto s : comb_) cudaStreamDestroy(s);
  for (auto e : events_) cudaEventDestroy(e);
  if (flags_) cudaFree(flags_);
  if (done_) cudaFree(done_);
  if (rounds_) cudaFree(rounds_);
  for (auto p : peer_slots_)
    if (p) cudaFree(p);
  if (impl_->stage) cudaFree(impl_->stage);
  delete impl_;
}

// Exchange (IPC handle, offset, layout key) of `local` with every rank (NCCL allgather on
// the dispatch communicator, blocking) and return each rank's pointer mapped here.
std::vector<char*> CeTransport::map_collective(const void* local, cudaStream_t s, uint64_t layout_key) {
  const int P = cm_->world;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (impl_->range_fn(&base, &size, (CUdeviceptr)local) != CUDA_SUCCESS)
    throw CudaError{"cuMemGetAddressRange failed"};
  cudaIpcMemHandle_t h;
  LINA_CUDA_CHECK(cudaIpcGetMemHandle(&h, (void*)base));
  unsigned char rec[128];
  std::memset(rec, 0, sizeof(rec));
  std::memcpy(rec, &h, sizeof(h));
  const uint64_t off = (uint64_t)((const char*)local - (const char*)base);
  std::memcpy(rec + 64, &off, 8);
  std::memcpy(rec + 72, &layout_key, 8);
  std::vector<unsigned char> all((size_t)128 * P);
  if (cm_->host_allgather) {  // host-bootstrap communicator: the caller's allgather
    LINA_CUDA_CHECK(cudaStreamSynchronize(s));
    host_allgather(cm_, rec, all.data(), 128);
  } else {
    char* st = (char*)impl_->stage;
    LINA_CUDA_CHECK(cudaMemcpyAsync(st + 128 * (size_t)cm_->rank, rec, 128, cudaMemcpyHostToDevice, s));
    LINA_NCCL_CHECK(ncclAllGather(st + 128 * (size_t)cm_->rank, st, 128, ncclUint8, cm_->ep_disp, s));
    LINA_CUDA_CHECK(cudaMemcpyAsync(all.data(), st, all.size(), cudaMemcpyDeviceToHost, s));
    LINA_CUDA_CHECK(cudaStreamSynchronize(s));
  }
  if (layout_key) {  // every rank sees the same records, so every rank throws or none does
    std::string bad;
    for (int r = 0; r < P; ++r) {
      uint64_t kr = 0;
      std::memcpy(&kr, all.data() + 128 * (size_t)r + 72, 8);
      if (kr != layout_key) bad += " " + std::to_string(r);
    }
    if (!bad.empty())
      throw ArgError{"peer-visible buffer layout differs on rank(s)" + bad +
                     ": capacity, n_chunks, num_experts, d_model, d_ffn, k and dtype must be equal on every "
                     "rank (inference: num_tokens too)"};
  }
  std::vector<char*> out(P, nullptr);
  for (int r = 0; r < P; ++r) {
    if (r == cm_->rank) {
      out[r] = (char*)local;
      continue;
    }
    cudaIpcMemHandle_t hr;
    std::memcpy(&hr, all.data() + 128 * (size_t)r, sizeof(hr));
    uint64_t offr = 0;
    std::memcpy(&offr, all.data() + 128 * (size_t)r + 64, 8);
    auto key = std::make_pair(r, std::string((const char*)&hr, sizeof(hr)));
    auto it = impl_->opened.find(key);
    char* mapped = nullptr;
    if (it != impl_->opened.end()) {
      mapped = it->second;
    } else {
      void* p = nullptr;
      LINA_CUDA_CHECK(cudaIpcOpenMemHandle(&p, hr, cudaIpcMemLazyEnablePeerAccess));
      mapped = (char*)p;
      impl_->opened[key] = mapped;
    }
    out[r] = mapped + offr;
  }
  return out;
}

const std::vector<char*>& CeTransport::peers(const void* local, cudaStream_t s, uint64_t layout_key) {
  const unsigned long long id = impl_->buffer_id(local);
  auto it = impl_->maps.find(local);
  if (it != impl_->maps.end() && it->second.buffer_id == id) return it->second.ptrs;
  Impl::Mapping m;
  m.ptrs = map_collective(local, s, layout_key);
  m.buffer_id = id;
  m.gen = ++impl_->next_gen;
  return (impl_->maps[local] = std::move(m)).ptrs;
}

uint64_t CeTransport::generation(const void* local) const {
  auto it = impl_->maps.find(local);
  return it == impl_->maps.end() ? 0 : it->second.gen;
}

uint32_t* const* CeTransport::peer_slots(int kind) {
  if (peer_slots_[kind]) return peer_slots_[kind];
  const int P = cm_->world;
  std::vector<uint32_t*> v(P);
  for (int r = 0; r < P; ++r) v[r] = (uint32_t*)peer_flags_[r] + slot(kind, cm_->rank, 0);
  void* d = nullptr;
  LINA_CUDA_CHECK(cudaMalloc(&d, sizeof(uint32_t*) * P));
  LINA_CUDA_CHECK(cudaMemcpy(d, v.data(), sizeof(uint32_t*) * P, cudaMemcpyHostToDevice));
  peer_slots_[kind] = (uint32_t**)d;
  return peer_slots_[kind];
}

void CeTransport::wait_flag(cudaStream_t s, int kind, int peer, int chunk, uint32_t value) {
  CUdeviceptr a = (CUdeviceptr)(flags_ + slot(kind, peer, chunk));
  if (impl_->wait_fn((CUstream)s, a, value, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
    throw CudaError{"cuStreamWaitValue32 failed"};
}

void CeTransport::post_flag(cudaStream_t s, int rank, int kind, int peer, int chunk, uint32_t value) {
  uint32_t* remote = (uint32_t*)peer_flags_[rank] + slot(kind, peer, chunk);
  if (impl_->write_fn((CUstream)s, (CUdeviceptr)remote, value, CU_STREAM_WRITE_VALUE_DEFAULT) !=
      CUDA_SUCCESS)
    throw CudaError{"cuStreamWriteValue32 failed"};
}

}  // namespace lina
