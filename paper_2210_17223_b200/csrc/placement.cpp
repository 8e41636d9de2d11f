// S10: popularity-driven expert replication (§5.2; §6.2).
//
// Eq. (1): n_e = N × popularity(e).  "For experts with the estimation n_e, we adopt
// the first-fit-decreasing heuristic to pack them into the empty devices so the
// total devices used are minimized"; experts with no estimate "are
// assigned evenly to the remaining free devices if any; otherwise are randomly
// assigned to a device"; "We set a maximum number of experts per
// device" (4 in the evaluation).
// Integerisation and tie rules are readings R14-R16.  The plan is a
// pure function of (popularity, N, max_per_device), so every rank computes the
// same tables with no broadcast.
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "layer.h"

namespace lina {

lina_status placement_compute(const double* pop, int E, int N, int mpd, lina_placement* out,
                              std::string* err) {
  if (E > N * mpd) {
    *err = "infeasible plan: " + std::to_string(E) + " experts > " + std::to_string(N) +
           " devices x " + std::to_string(mpd) + " per device";
    return LINA_ERR_INFEASIBLE_PLAN;
  }
  // Eq. (1) and integer replica counts r_e = max(1, round-half-up(n_e)), r_e <= N.
  std::vector<double> ne(E);
  std::vector<int> r(E);
  for (int e = 0; e < E; ++e) {
    ne[e] = (double)N * pop[e];
    int re = (int)std::floor(ne[e] + 0.5);
    r[e] = std::min(N, std::max(1, re));
  }
  long total = 0;
  for (int e = 0; e < E; ++e) total += r[e];
  while (total > (long)N * mpd) {  // trim the largest count (ties: larger id) first
    int best = -1;
    for (int e = 0; e < E; ++e)
      if (best < 0 || r[e] >= r[best]) best = e;
    r[best] -= 1;
    --total;
  }
  struct Item {
    double size;
    int e, q;
  };
  std::vector<Item> items;
  for (int e = 0; e < E; ++e)
    for (int q = 0; q < r[e]; ++q) items.push_back({ne[e] / r[e], e, q});
  std::sort(items.begin(), items.end(), [](const Item& a, const Item& b) {
    if (a.size != b.size) return a.size > b.size;
    if (a.e != b.e) return a.e < b.e;
    return a.q < b.q;
  });
  std::vector<double> load(N, 0.0);
  std::vector<std::vector<int>> hosted(N);
  const double eps = 1e-9;
  for (const Item& it : items) {
    int first_fit = -1, least = -1;
    for (int dv = 0; dv < N; ++dv) {
      if ((int)hosted[dv].size() >= mpd) continue;
      if (std::find(hosted[dv].begin(), hosted[dv].end(), it.e) != hosted[dv].end()) continue;
      if (first_fit < 0 && load[dv] + it.size <= 1.0 + eps) first_fit = dv;
      if (least < 0 || load[dv] < load[least]) least = dv;
    }
    const int dv = first_fit >= 0 ? first_fit : least;
    if (dv < 0) {
      *err = "infeasible plan: no device can host another replica of expert " + std::to_string(it.e);
      return LINA_ERR_INFEASIBLE_PLAN;
    }
    load[dv] += it.size;
    hosted[dv].push_back(it.e);
  }
  out->num_experts = E;
  out->num_devices = N;
  out->max_per_device = mpd;
  for (int e = 0; e < E; ++e) {
    out->replicas[e] = r[e];
    int q = 0;
    for (int dv = 0; dv < N; ++dv)
      if (std::find(hosted[dv].begin(), hosted[dv].end(), e) != hosted[dv].end())
        out->replica_device[(size_t)e * out->max_replicas + q++] = dv;
    for (; q < out->max_replicas; ++q) out->replica_device[(size_t)e * out->max_replicas + q] = -1;
  }
  for (int dv = 0; dv < N; ++dv) {
    std::sort(hosted[dv].begin(), hosted[dv].end());
    for (int i = 0; i < mpd; ++i)
      out->hosted[(size_t)dv * mpd + i] = i < (int)hosted[dv].size() ? hosted[dv][i] : -1;
  }
  return LINA_OK;
}

// Tokens of one (source, expert) pair per replica: contiguous blocks in slot order,
// sizes differing by <= 1; block q goes to replica (q + source_rank) mod r (R14).
void replica_split(int count, int replicas, int source_rank, int* out) {
  const int base = count / replicas, extra = count % replicas;
  for (int i = 0; i < replicas; ++i) out[i] = 0;
  for (int q = 0; q < replicas; ++q) out[(q + source_rank) % replicas] += base + (q < extra ? 1 : 0);
}

}  // namespace lina
