// Internal entry points between api.cpp, layer.cpp, infer.cpp and sched.cpp.
#pragma once
#include "internal.h"
#include "kernels.h"

#include <deque>
#include <string>
#include <unordered_map>
#include <vector>

// One profiled distribution Ψ: per-expert selection counts, their total, and its top-k
// experts (count desc, id asc) with P = count / total — refreshed by every add.
struct PathDist {
  std::vector<int64_t> c;
  int64_t total = 0;
  std::vector<int32_t> top;
  std::vector<double> prob;
};

// Packed path -> PathDist: open addressing with linear probing over a power-of-two key
// array (one cache line per probe, instead of a node chase per bucket).  Entries live in
// a deque, so references stay valid while the table grows.
class FlatPathMap {
 public:
  PathDist& operator[](uint64_t key) {
    if ((n_ + 1) * 2 > keys_.size()) grow();
    size_t i = slot_of(key);
    if (idx_[i] < 0) {
      idx_[i] = (int32_t)dists_.size();
      keys_[i] = key;
      dists_.emplace_back();
      dist_keys_.push_back(key);
      ++n_;
    }
    return dists_[(size_t)idx_[i]];
  }
  const PathDist* find(uint64_t key) const {
    if (keys_.empty()) return nullptr;
    const size_t i = slot_of(key);
    return idx_[i] < 0 ? nullptr : &dists_[(size_t)idx_[i]];
  }
  size_t size() const { return n_; }
  template <typename F>
  void for_each(F f) const {
    for (size_t j = 0; j < dists_.size(); ++j) f(dist_keys_[j], dists_[j]);
  }

 private:
  static uint64_t mix(uint64_t x) {  // splitmix64 finaliser: packed keys are far from uniform
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    return x ^ (x >> 31);
  }
  size_t slot_of(uint64_t key) const {  // the key's slot, or the empty slot where it belongs
    const size_t mask = keys_.size() - 1;
    size_t i = (size_t)mix(key) & mask;
    while (idx_[i] >= 0 && keys_[i] != key) i = (i + 1) & mask;
    return i;
  }
  void grow() {
    const size_t cap = keys_.empty() ? 64 : keys_.size() * 2;
    keys_.assign(cap, 0);
    idx_.assign(cap, -1);
    for (size_t j = 0; j < dist_keys_.size(); ++j) {
      const size_t i = slot_of(dist_keys_[j]);
      keys_[i] = dist_keys_[j];
      idx_[i] = (int32_t)j;
    }
  }
  std::vector<uint64_t> keys_;
  std::vector<int32_t> idx_;
  std::deque<PathDist> dists_;
  std::vector<uint64_t> dist_keys_;
  size_t n_ = 0;
};

// Sample-path popularity profile (popularity.cpp; paper D4: host DRAM).
struct lina_pop_profile {
  int L = 0, E = 0, k = 0, l = 0;
  int bits = 0;         // bits per expert id in a packed key
  bool packed = false;  // l·k·bits <= 64: paths are uint64 keys, else byte strings
  // [m * (l + 1) + s] for 1 <= s <= min(l, m): path (s sorted expert sets) -> per-expert
  // selection counts in layer m
  std::vector<FlatPathMap> maps64;
  std::vector<std::unordered_map<std::string, PathDist>> maps;
  std::vector<PathDist> marg;  // [L] layer marginals (backoff)
};

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
// (all three are no-ops while `s` is being captured into a CUDA graph: the scheduler tracks
// eagerly launched all-to-all phases; a captured event would never be recorded)
void sched_a2a_imminent(lina_comm* cm, cudaStream_t s);   // combine-bwd started
void sched_a2a_begin(lina_comm* cm, cudaStream_t a2a_stream);
void sched_a2a_end(lina_comm* cm, cudaStream_t a2a_stream);  // phase ends there

Scheduler* sched_create(lina_comm* cm);
void sched_destroy(Scheduler* s);
void sched_config(Scheduler* s, lina_policy p, size_t partition_bytes);
void sched_submit(Scheduler* s, void* grad, size_t count, lina_dtype dt, cudaStream_t ready);
void sched_wait(Scheduler* s, cudaStream_t st);  // device-side wait point, host never blocks
void sched_check(Scheduler* s);                  // rethrows an error of the scheduler thread
void sched_stats(Scheduler* s, int64_t* issued, int64_t* deferred);

// Expert packing (packing.cpp).
int pack_decide(int world, int pack, double ffn_ms, double a2a_ms);
void pack_weights(lina_comm* cm, int E, int m0, int m1, size_t expert_bytes, const void* w_from, void* w_to,
                  cudaStream_t s);

// Placement (placement.cpp).
lina_status placement_compute(const double* pop, int E, int N, int mpd, lina_placement* out,
                              std::string* err);
void replica_split(int count, int replicas, int source_rank, int* out);

// Popularity estimation / two-phase scheduling (popularity.cpp).
lina_pop_profile* popprof_create(int L, int E, int k, int l);
std::string popprof_check_ids(const lina_pop_profile* p, const int32_t* sel, int64_t rows, int layers);
void popprof_add(lina_pop_profile* p, const int32_t* sel, int64_t T);
void popprof_estimate(const lina_pop_profile* p, int m, const int32_t* hist, int64_t T, double* pop,
                      int32_t* topk);
bool phase_two_identical(const double* est, const int32_t* actual, int E, int k);
std::string popprof_save(const lina_pop_profile* p, const char* path);   // "" or the error
std::string popprof_load(const char* path, lina_pop_profile** out);      // "" or the error

}  // namespace lina
