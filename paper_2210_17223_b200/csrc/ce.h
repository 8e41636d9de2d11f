// Copy-engine all-to-all transport (ce.cpp).
#pragma once
#include <map>
#include <string>
#include <vector>

#include "internal.h"

namespace lina {

class CeTransport {
 public:
  // flag kinds: READY (at the receiver) and PULLED (at the sender) per exchange
  enum { kReadyFwdD = 0, kReadyFwdC = 1, kReadyBwdD = 2, kReadyBwdC = 3,
         kPulledFwdD = 4, kPulledFwdC = 5, kPulledBwdD = 6, kPulledBwdC = 7,
         kFreeFwd = 8, kFreeBwd = 9,
         // fused transport (in-kernel signals; rounds from the device counters below)
         kFReadyFwdD = 10, kFReadyFwdC = 11, kFReadyBwdD = 12, kFReadyBwdC = 13,
         // inference exchange by peer stores (infer.cpp)
         kIFreeD = 14, kIReadyD = 15, kIFreeC = 16, kIReadyC = 17,
         // dropless training: the per-expert counts of a forward have landed
         kFCountFwd = 18,
         // split dispatch (n = 1): a forward's per-expert counts have landed (before the rows)
         kFCountFwdS = 19, kKinds = 20 };
  static constexpr int kMaxChunks = 32;

  explicit CeTransport(lina_comm* cm);  // collective (allgathers the flag-array handles)
  ~CeTransport();
  // Every rank's copy of `local` (same offset in its own buffer), mapped into this
  // process; collective on the first call for an allocation, cached afterwards.  The
  // cache is keyed by the pointer AND the allocation's process-wide buffer id, so a
  // buffer freed and re-allocated at the same address is mapped again (collectively:
  // every rank passes its new buffers in the same call, as an SPMD program does) instead
  // of reusing a stale peer mapping.  layout_key != 0: every rank must map this buffer
  // with the same key (a hash of the peer-visible layout), else ArgError on every rank.
  const std::vector<char*>& peers(const void* local, cudaStream_t s, uint64_t layout_key = 0);
  // Mapping generation of `local` (changes whenever peers() re-maps it; 0 = unmapped).
  uint64_t generation(const void* local) const;
  // Stream `s` waits until my flag (kind, peer, chunk) >= value.
  void wait_flag(cudaStream_t s, int kind, int peer, int chunk, uint32_t value);
  // Stream `s` writes `value` into rank `rank`'s flag (kind, peer, chunk).
  void post_flag(cudaStream_t s, int rank, int kind, int peer, int chunk, uint32_t value);
  // Device array of the P pointers peers(local)[r] + offset (cached; uploaded once).
  void* const* dev_ptrs(const void* local, size_t offset, cudaStream_t s, uint64_t layout_key = 0);
  // In-kernel signalling (signal.h): my slots of `kind` (peer r at r * kMaxChunks), the
  // device array [P] of every rank's slot (kind, me) mapped here (uploaded once), and a
  // zeroed CTA-completion counter per call site (sites < kDoneSites).
  const uint32_t* slots(int kind) const { return flags_ + slot(kind, 0, 0); }
  uint32_t* const* peer_slots(int kind);
  unsigned int* done_counter(int site) const { return done_ + site; }
  // device round counters of the fused transport: [0] forward, [1] backward
  uint32_t* round_fwd() const { return rounds_; }
  uint32_t* round_bwd() const { return rounds_ + 1; }
  uint32_t* round_inf() const { return rounds_ + 2; }
  static constexpr int kDoneSites = 32;  // 16..23 / 24..31: split dispatch, per owner block
  cudaStream_t disp_stream(int peer) const { return disp_[peer]; }
  cudaStream_t comb_stream(int peer) const { return comb_[peer]; }
  // event pool: [which (0..3)][peer][chunk or kMaxChunks(+1)]
  cudaEvent_t ev(int which, int peer, int chunk) const {
    return events_[((size_t)which * cm_->world + peer) * (kMaxChunks + 2) + chunk];
  }
  // host-side cache of per-rank tensor-map arrays (fused transport epilogue stores)
  std::map<std::string, std::vector<unsigned char>> host_blobs;
  uint32_t seq_fwd = 0, seq_bwd = 0;
  // rounds that ran the copy-engine pipeline (its PULLED flags carry these values)
  uint32_t last_ce_fwd = 0, last_ce_bwd = 0, prev_ce_fwd = 0, prev_ce_bwd = 0;

 private:
  size_t slot(int kind, int peer, int chunk) const {
    return ((size_t)kind * cm_->world + peer) * kMaxChunks + chunk;
  }
  std::vector<char*> map_collective(const void* local, cudaStream_t s, uint64_t layout_key);
  lina_comm* cm_;
  struct Impl;
  Impl* impl_;
  uint32_t* flags_ = nullptr;
  size_t nflags_ = 0;
  unsigned int* done_ = nullptr;
  uint32_t* rounds_ = nullptr;
  std::vector<uint32_t**> peer_slots_;
  std::vector<char*> peer_flags_;
  std::vector<cudaStream_t> disp_, comb_;
  std::vector<cudaEvent_t> events_;
};

}  // namespace lina
