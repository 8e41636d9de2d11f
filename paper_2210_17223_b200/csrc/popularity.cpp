// Popularity estimation and two-phase scheduling (§5.2).
//
// "We then group tokens that select the same experts from layer i-l to layer i, which
// represent a unique sample path of experts used.  For each sample path j, we compute
// the expert popularity distribution Ψ_j^{i+1} for layer i+1".  "For a
// sample path j, we pick the top-k expert(s) of the subsequent layer from Ψ_j^{i+1}
// and use their probabilities {P_j^{i+1}(e)}"; Eq. (1) aggregates
// Σ_t P_{j(t)}(e) / N_t.  Phase two compares "the overall top-2k experts"
// (P:482-484).  Profiles live in host DRAM as hash maps per layer (paper D4).
// Readings R19-R22.
//
// Layout: per target layer m and path length s, one hash map keyed by the path's expert
// sets (each sorted ascending) -> per-expert counts.  Keys are the ids bit-packed into a
// uint64 when l·k·ceil(log2 E) <= 64 (every config here), else s·k int32 byte strings.
// Every entry keeps its top-k and P (refreshed by each add), so an estimate is one hash
// lookup per backoff level and k additions per token; counts are integers, so the
// distribution chosen and the per-token P are exact functions of the trace.
#include <algorithm>
#include <memory>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "layer.h"

namespace lina {

namespace {

// One token's selections in one layer as a sorted set (R19), into v[0..k).
const int32_t* sorted_set(const int32_t* sel, int k, int32_t* tmp, std::vector<int32_t>* big) {
  int32_t* v = tmp;
  if (k > 64) {
    big->resize(k);
    v = big->data();
  }
  std::memcpy(v, sel, sizeof(int32_t) * k);
  std::sort(v, v + k);
  return v;
}

// Key of the path made of the s layer rows rows[0..s) (each k ids): bit-packed or bytes.
struct PathKey {
  const lina_pop_profile* p;
  uint64_t u = 0;
  std::string str;
  int32_t tmp[64];
  std::vector<int32_t> big;
  void build(const int32_t* rows, int s) {
    const int k = p->k;
    u = 0;
    str.clear();
    for (int i = 0; i < s; ++i) {
      const int32_t* v = sorted_set(rows + (int64_t)i * k, k, tmp, &big);
      if (p->packed)
        for (int q = 0; q < k; ++q) u = (u << p->bits) | (uint64_t)v[q];
      else
        str.append(reinterpret_cast<const char*>(v), sizeof(int32_t) * k);
    }
  }
  PathDist& slot(lina_pop_profile* pp, size_t map) {
    return pp->packed ? pp->maps64[map][u] : pp->maps[map][str];
  }
  const PathDist* find(size_t map) const {
    if (p->packed) {
      return p->maps64[map].find(u);
    }
    auto it = p->maps[map].find(str);
    return it == p->maps[map].end() ? nullptr : &it->second;
  }
};

// k experts with the largest counts, ties to the lower id (R21).
void top_k(const std::vector<int64_t>& c, int k, std::vector<int>* out) {
  const int E = (int)c.size();
  if (k <= 8) {  // k linear passes: the first strict maximum not yet taken
    out->clear();
    for (int q = 0; q < k; ++q) {
      int best = -1;
      for (int e = 0; e < E; ++e) {
        if (best >= 0 && c[e] <= c[best]) continue;
        if (std::find(out->begin(), out->end(), e) != out->end()) continue;
        best = e;
      }
      out->push_back(best);
    }
    return;
  }
  out->resize(E);
  for (int e = 0; e < E; ++e) (*out)[e] = e;
  std::partial_sort(out->begin(), out->begin() + k, out->end(), [&](int a, int b) {
    return c[a] != c[b] ? c[a] > c[b] : a < b;
  });
  out->resize(k);
}

// Recompute a distribution's total, top-k and P after its counts changed (R20, R21).
void refresh(PathDist* d, int k) {
  d->total = 0;
  for (int64_t x : d->c) d->total += x;
  std::vector<int> chosen;
  top_k(d->c, k, &chosen);
  d->top.assign(chosen.begin(), chosen.end());
  d->prob.resize(k);
  for (int q = 0; q < k; ++q) d->prob[q] = d->total ? (double)d->c[chosen[q]] / (double)d->total : 0.0;
}

}  // namespace

std::string popprof_check_ids(const lina_pop_profile* p, const int32_t* sel, int64_t rows, int layers) {
  for (int64_t t = 0; t < rows; ++t)
    for (int i = 0; i < layers; ++i) {
      const int32_t* s = sel + (t * layers + i) * p->k;
      for (int q = 0; q < p->k; ++q) {
        if (s[q] < 0 || s[q] >= p->E)
          return "token " + std::to_string(t) + " layer slot " + std::to_string(i) + ": expert id " +
                 std::to_string(s[q]) + " outside [0, " + std::to_string(p->E) + ")";
        for (int r = 0; r < q; ++r)
          if (s[r] == s[q])
            return "token " + std::to_string(t) + " layer slot " + std::to_string(i) +
                   " selects expert " + std::to_string(s[q]) + " twice";
      }
    }
  return "";
}

lina_pop_profile* popprof_create(int L, int E, int k, int l) {
  auto* p = new lina_pop_profile;
  p->L = L;
  p->E = E;
  p->k = k;
  p->l = l;
  int bits = 1;
  while ((1 << bits) < E) ++bits;
  p->bits = bits;
  p->packed = (int64_t)l * k * bits <= 64;
  if (p->packed) p->maps64.resize((size_t)L * (l + 1));
  else p->maps.resize((size_t)L * (l + 1));
  p->marg.resize(L);
  for (auto& d : p->marg) {
    d.c.assign(E, 0);
    refresh(&d, k);
  }
  return p;
}

void popprof_add(lina_pop_profile* p, const int32_t* sel, int64_t T) {
  const int L = p->L, k = p->k, l = p->l;
  PathKey key{p};
  std::vector<PathDist*> touched;  // entries whose summary must be refreshed
  for (int64_t t = 0; t < T; ++t) {
    const int32_t* st = sel + t * (int64_t)L * k;
    for (int m = 0; m < L; ++m) {
      const int32_t* next = st + (int64_t)m * k;
      for (int q = 0; q < k; ++q) p->marg[m].c[next[q]] += 1;
      for (int s = 1; s <= std::min(l, m); ++s) {
        key.build(st + (int64_t)(m - s) * k, s);
        PathDist& d = key.slot(p, (size_t)m * (l + 1) + s);
        if (d.c.empty()) d.c.assign(p->E, 0);
        if (d.total >= 0) {  // first touch in this call (refresh sets total >= 0 again)
          d.total = -1;
          touched.push_back(&d);
        }
        for (int q = 0; q < k; ++q) d.c[next[q]] += 1;
      }
    }
  }
  for (PathDist* d : touched) refresh(d, k);
  if (T > 0)
    for (auto& d : p->marg) refresh(&d, k);
}

// The distribution Ψ is read from for one token's history (R20): the longest seen
// suffix, else the layer marginal; nullptr when neither has any selection.
static const PathDist* distribution(const lina_pop_profile* p, int m, const int32_t* hist, PathKey* key) {
  const int k = p->k, l = p->l;
  if (p->packed) {  // the length-s suffix of a packed path is its low s·k·bits bits
    key->build(hist, l);
    const uint64_t full = key->u;
    for (int s = l; s >= 1; --s) {
      const int nb = s * k * p->bits;
      key->u = nb >= 64 ? full : (full & ((uint64_t(1) << nb) - 1));
      if (const PathDist* d = key->find((size_t)m * (l + 1) + s)) return d;
    }
  } else {
    for (int s = l; s >= 1; --s) {
      key->build(hist + (int64_t)(l - s) * k, s);
      if (const PathDist* d = key->find((size_t)m * (l + 1) + s)) return d;
    }
  }
  return p->marg[m].total > 0 ? &p->marg[m] : nullptr;
}

void popprof_estimate(const lina_pop_profile* p, int m, const int32_t* hist, int64_t T, double* pop,
                      int32_t* topk) {
  const int E = p->E, k = p->k, l = p->l;
  std::vector<double> acc(E, 0.0);
  PathKey key{p};
  for (int64_t t = 0; t < T; ++t) {
    const PathDist* d = distribution(p, m, hist + t * (int64_t)l * k, &key);
    for (int q = 0; q < k; ++q) {
      if (d) acc[d->top[q]] += d->prob[q];  // P_j(e) = Ψ_j(e), summed in token order (Eq. (1))
      if (topk) topk[t * k + q] = d ? d->top[q] : -1;
    }
  }
  for (int e = 0; e < E; ++e) pop[e] = T ? acc[e] / (double)T : 0.0;
}

// ---- persistence: "LINAPOP1", int32 L E k l, int8 packed, marginals [L][E] int64, then per
// map (in index order) int64 n_entries and n × (key, counts[E] int64); a packed key is a
// uint64, a string key an int32 byte length + bytes.
namespace {
struct File {
  FILE* f;
  explicit File(FILE* x) : f(x) {}
  ~File() {
    if (f) fclose(f);
  }
};
template <typename T>
bool put(FILE* f, const T& v) { return fwrite(&v, sizeof(T), 1, f) == 1; }
template <typename T>
bool get(FILE* f, T* v) { return fread(v, sizeof(T), 1, f) == 1; }
bool put_counts(FILE* f, const std::vector<int64_t>& c) {
  return fwrite(c.data(), sizeof(int64_t), c.size(), f) == c.size();
}
bool get_counts(FILE* f, std::vector<int64_t>* c, int E) {
  c->resize(E);
  if (fread(c->data(), sizeof(int64_t), E, f) != (size_t)E) return false;
  for (int64_t x : *c)
    if (x < 0) return false;
  return true;
}
}  // namespace

std::string popprof_save(const lina_pop_profile* p, const char* path) {
  File fh(fopen(path, "wb"));
  FILE* f = fh.f;
  if (!f) return std::string("cannot open ") + path + " for writing";
  bool ok = fwrite("LINAPOP1", 1, 8, f) == 8 && put<int32_t>(f, p->L) && put<int32_t>(f, p->E) &&
            put<int32_t>(f, p->k) && put<int32_t>(f, p->l) && put<int8_t>(f, p->packed ? 1 : 0);
  for (int m = 0; ok && m < p->L; ++m) ok = put_counts(f, p->marg[m].c);
  const size_t nmaps = (size_t)p->L * (p->l + 1);
  for (size_t i = 0; ok && i < nmaps; ++i) {
    if (p->packed) {
      ok = put<int64_t>(f, (int64_t)p->maps64[i].size());
      p->maps64[i].for_each([&](uint64_t key, const PathDist& d) {
        if (ok) ok = put<uint64_t>(f, key) && put_counts(f, d.c);
      });
    } else {
      ok = put<int64_t>(f, (int64_t)p->maps[i].size());
      for (const auto& kv : p->maps[i]) {
        if (!ok) break;
        ok = put<int32_t>(f, (int32_t)kv.first.size()) &&
             fwrite(kv.first.data(), 1, kv.first.size(), f) == kv.first.size() && put_counts(f, kv.second.c);
      }
    }
  }
  if (!ok) return std::string("write to ") + path + " failed";
  return "";
}

std::string popprof_load(const char* path, lina_pop_profile** out) {
  File fh(fopen(path, "rb"));
  FILE* f = fh.f;
  if (!f) return std::string("cannot open ") + path;
  char magic[8];
  int32_t L, E, k, l;
  int8_t packed;
  if (fread(magic, 1, 8, f) != 8 || std::memcmp(magic, "LINAPOP1", 8) != 0) return "not a LINAPOP1 file";
  if (!get(f, &L) || !get(f, &E) || !get(f, &k) || !get(f, &l) || !get(f, &packed)) return "truncated header";
  if (L < 2 || E < 1 || k < 1 || k > E || l < 1 || l >= L) return "invalid shape in header";
  std::unique_ptr<lina_pop_profile> p(popprof_create(L, E, k, l));
  if ((packed != 0) != p->packed) return "key layout does not match the shape";
  for (int m = 0; m < L; ++m) {
    if (!get_counts(f, &p->marg[m].c, E)) return "truncated or negative marginals";
    refresh(&p->marg[m], k);
  }
  const size_t nmaps = (size_t)L * (l + 1);
  const int32_t key_bytes_max = (int32_t)(sizeof(int32_t) * (size_t)l * k);
  for (size_t i = 0; i < nmaps; ++i) {
    int64_t n;
    if (!get(f, &n) || n < 0) return "truncated map header";
    for (int64_t j = 0; j < n; ++j) {
      std::vector<int64_t> c;
      if (p->packed) {
        uint64_t key;
        if (!get(f, &key) || !get_counts(f, &c, E)) return "truncated map entry";
        PathDist& d = p->maps64[i][key];
        d.c = std::move(c);
        refresh(&d, k);
      } else {
        int32_t len;
        if (!get(f, &len) || len < 0 || len > key_bytes_max) return "bad key length";
        std::string key((size_t)len, '\0');
        if (fread(&key[0], 1, (size_t)len, f) != (size_t)len || !get_counts(f, &c, E)) return "truncated map entry";
        PathDist& d = p->maps[i][key];
        d.c = std::move(c);
        refresh(&d, k);
      }
    }
  }
  *out = p.release();
  return "";
}

bool phase_two_identical(const double* est, const int32_t* actual, int E, int k) {
  const int n = std::min(E, 2 * k);
  std::vector<int> a(E), b(E);
  for (int e = 0; e < E; ++e) a[e] = b[e] = e;
  std::partial_sort(a.begin(), a.begin() + n, a.end(),
                    [&](int x, int y) { return est[x] != est[y] ? est[x] > est[y] : x < y; });
  std::partial_sort(b.begin(), b.begin() + n, b.end(),
                    [&](int x, int y) { return actual[x] != actual[y] ? actual[x] > actual[y] : x < y; });
  std::sort(a.begin(), a.begin() + n);
  std::sort(b.begin(), b.begin() + n);
  return std::equal(a.begin(), a.begin() + n, b.begin());
}

}  // namespace lina
