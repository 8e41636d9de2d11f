// In-kernel cross-rank ordering for the fused transport (internal header).
//
// A rank's flag slot (kind, peer) lives in its IPC-mapped flag array (ce.cpp); rank r
// publishes "my part of exchange `kind` of round `seq` is done" by a release store of
// seq into every peer's slot (kind, r), and a consumer kernel acquires it by spinning
// (one thread per CTA) until every peer's slot reached the round it needs.  This
// replaces one stream wait / stream write operation per peer and exchange (~6 us of
// device time each, measured) by a few loads inside kernels that run anyway.
//
//   wait side : thread 0 of each CTA calls sig_wait() before the CTA touches data the
//               peers wrote (then __syncthreads; a TMA consumer adds a proxy fence).
//   post side : sig_post() by one thread when only it has to publish (nothing written
//               yet by the kernel), or sig_post_last() by thread 0 of every CTA after
//               its last write: the last CTA to finish publishes for the whole grid.
//
// A peer that never posts must not hang the GPU: a waiter traps after ~10 s.
#pragma once
#include <stdint.h>

namespace lina {

// Rounds live in device memory, one forward and one backward counter per rank: during a
// pass every signal carries counter + 1, and the pass's last kernel bumps the counter
// (last CTA).  So every pass has its own round (interleaved layers sharing a comm stay
// ordered), and the kernels — and a CUDA graph captured around them — carry pointers,
// not round numbers.
struct PeerSignal {
  const uint32_t* wait = nullptr;        // my slots of the awaited kind: wait[r * stride] written by rank r
  const uint32_t* wait_round = nullptr;  // wait until every peer's slot >= *wait_round + wait_add (wrap-safe)
  uint32_t wait_add = 0;
  uint32_t* const* post = nullptr;       // device array [P]: rank r's slot (kind, me), mapped here
  const uint32_t* post_round = nullptr;  // publish *post_round + post_add
  uint32_t post_add = 0;
  uint32_t* bump = nullptr;              // sig_bump_last(): the pass's round counter
  unsigned int* done = nullptr;          // zeroed CTA-completion counter (sig_post_last / sig_bump_last)
  int P = 1, me = 0, stride = 0;
  int wait_chunks = 1;                   // micro-op slots wait[r*stride + 0 .. wait_chunks-1] per peer
  int post_chunk = 0;                    // micro-op slot published: post[r] + post_chunk
};

#ifdef __CUDACC__
__device__ __forceinline__ uint32_t sig_ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void sig_st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void sig_wait(const PeerSignal& s) {
  if (!s.wait) return;
  const uint32_t target = *s.wait_round + s.wait_add;
  const long long t0 = clock64();
  for (int r = 0; r < s.P; ++r) {
    if (r == s.me) continue;
    for (int c = 0; c < s.wait_chunks; ++c) {
      const uint32_t* f = s.wait + (size_t)r * s.stride + c;
      while ((int)(sig_ld_acquire(f) - target) < 0) {
        __nanosleep(100);
        if (clock64() - t0 > 20000000000LL) __trap();  // a peer died: fail loudly, do not hang
      }
    }
  }
}

__device__ __forceinline__ void sig_post(const PeerSignal& s) {
  if (!s.post) return;
  const uint32_t v = *s.post_round + s.post_add;
  __threadfence_system();
  for (int r = 0; r < s.P; ++r)
    if (r != s.me) sig_st_release(s.post[r] + s.post_chunk, v);
}

// The CTA's writes (ordered before thread 0 by the caller's barrier) are released to the
// last CTA at GPU scope; only that CTA pays the system-scope fence before publishing
// (release/acquire chains compose: a peer that acquires the flag sees every CTA's writes).
__device__ __forceinline__ void sig_post_last(const PeerSignal& s) {
  if (!s.post) return;
  const unsigned int nb = gridDim.x * gridDim.y * gridDim.z;
  unsigned int prev;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(s.done) : "memory");
  if (prev == nb - 1) {
    *s.done = 0u;  // reset for the next launch on this stream
    sig_post(s);
  }
}

// Wait for one peer's slots only (the split dispatch: a consumer takes the rows of source
// r as soon as r has posted them).
__device__ __forceinline__ void sig_wait_one(const PeerSignal& s, int r) {
  if (!s.wait || r == s.me) return;
  const uint32_t target = *s.wait_round + s.wait_add;
  const long long t0 = clock64();
  for (int c = 0; c < s.wait_chunks; ++c) {
    const uint32_t* f = s.wait + (size_t)r * s.stride + c;
    while ((int)(sig_ld_acquire(f) - target) < 0) {
      __nanosleep(64);
      if (clock64() - t0 > 20000000000LL) __trap();
    }
  }
}

// Thread 0 of every CTA after its last store to `owner`: the last of the `nb` CTAs
// publishes READY to that owner alone (`done` = that owner's zeroed counter).
__device__ __forceinline__ void sig_post_owner_last(const PeerSignal& s, unsigned int* done, int owner,
                                                    unsigned int nb) {
  if (!s.post) return;
  unsigned int prev;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(done) : "memory");
  if (prev == nb - 1) {
    *done = 0u;
    const uint32_t v = *s.post_round + s.post_add;
    __threadfence_system();
    sig_st_release(s.post[owner] + s.post_chunk, v);
  }
}

// Thread 0 of every CTA, after its last use of the round: the last CTA closes the round.
__device__ __forceinline__ void sig_bump_last(const PeerSignal& s) {
  if (!s.bump) return;
  const unsigned int nb = gridDim.x * gridDim.y * gridDim.z;
  unsigned int prev;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(s.done) : "memory");
  if (prev == nb - 1) {
    *s.done = 0u;
    *s.bump = *s.bump + 1u;
  }
}
#endif

}  // namespace lina
