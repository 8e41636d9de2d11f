// Diagnostic phase trace (LINA_TRACE=1 at comm init): events recorded on the layer's
// stream at phase boundaries; the deltas between consecutive marks of one call are
// accumulated (resolved lazily at the next call) and printed per rank at comm destroy.
// Off by default; never on a timed path of bench.py.
#include <algorithm>
#include <cstdio>
#include <map>
#include <string>
#include <vector>

#include "common.h"
#include "internal.h"

namespace lina {

struct Trace {
  using Group = std::vector<std::pair<std::string, cudaEvent_t>>;  // the marks of one call
  std::vector<Group> groups;
  std::vector<cudaEvent_t> pool;
  std::map<std::string, std::vector<float>> acc;
  std::vector<std::string> order;
};

Trace* trace_create() { return new Trace(); }

void trace_mark(lina_comm* cm, cudaStream_t s, const char* label) {
  Trace* t = cm->trace;
  if (!t) return;
  if (t->groups.empty()) t->groups.emplace_back();
  cudaEvent_t e;
  if (t->pool.empty()) {
    LINA_CUDA_CHECK(cudaEventCreate(&e));
  } else {
    e = t->pool.back();
    t->pool.pop_back();
  }
  LINA_CUDA_CHECK(cudaEventRecord(e, s));
  t->groups.back().push_back({label, e});
}

static void accumulate(Trace* t, Trace::Group& g) {
  for (size_t i = 1; i < g.size(); ++i) {
    float ms = 0.f;
    LINA_CUDA_CHECK(cudaEventElapsedTime(&ms, g[i - 1].second, g[i].second));
    const std::string key = g[i - 1].first + " -> " + g[i].first;
    auto it = t->acc.find(key);
    if (it == t->acc.end()) {
      t->order.push_back(key);
      t->acc[key] = {ms};
    } else {
      it->second.push_back(ms);
    }
  }
  for (auto& pe : g) t->pool.push_back(pe.second);
  g.clear();
}

// Called at the start of every layer call: opens a new group and folds in the earlier
// groups whose last mark has completed (never blocks, so the trace does not serialise
// the host with the device).
void trace_flush(lina_comm* cm) {
  Trace* t = cm->trace;
  if (!t) return;
  std::vector<Trace::Group> keep;
  for (auto& g : t->groups) {
    if (g.empty()) continue;
    if (cudaEventQuery(g.back().second) == cudaSuccess) {
      accumulate(t, g);
    } else {
      (void)cudaGetLastError();  // clear cudaErrorNotReady
      keep.push_back(std::move(g));
    }
  }
  keep.emplace_back();
  t->groups = std::move(keep);
}

void trace_destroy(lina_comm* cm) {
  Trace* t = cm->trace;
  if (!t) return;
  try {
    cudaDeviceSynchronize();
    for (auto& g : t->groups)
      if (!g.empty()) accumulate(t, g);
  } catch (...) {
  }
  for (const auto& k : t->order) {
    std::vector<float> v = t->acc[k];
    std::sort(v.begin(), v.end());
    std::fprintf(stderr, "[lina trace rank %d] %-36s median %8.2f us  min %8.2f  max %9.2f  (n=%zu)\n", cm->rank,
                 k.c_str(), 1e3 * v[v.size() / 2], 1e3 * v.front(), 1e3 * v.back(), v.size());
  }
  for (auto e : t->pool) cudaEventDestroy(e);
  delete t;
  cm->trace = nullptr;
}

}  // namespace lina
