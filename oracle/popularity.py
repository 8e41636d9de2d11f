"""Oracle for popularity estimation and two-phase scheduling — TEST INFRASTRUCTURE ONLY.

(See oracle/__init__.py: only tests/, smoke() and bench.py's CPU legs may import this.)

PAPER.md §5.2 (A17, A20, D4):
  "In the profiling stage, we collect the expert selection results of all tokens ...
  We then group tokens that select the same experts from layer i-l to layer i, which
  represent a unique sample path of experts used.  For each sample path j, we compute
  the expert popularity distribution Ψ_j^{i+1} for layer i+1".
  "In each layer i, for a sample path j, we pick the top-k expert(s) of the subsequent
  layer from Ψ_j^{i+1} and use their probabilities {P_j^{i+1}(e)} to represent expert
  popularity"; Eq. (1) then uses "Σ_{t=1}^{N_t} P^{i+1}_{j(t)}(e)/N_t"
  as the overall popularity of expert e.
  Phase two: "comparing the overall top-2k experts.  If the two lists are identical, no
  fine-tuning is needed ... Otherwise, the scheduler re-computes the resource
  allocation with the actual expert popularity".

Readings (R19-R22):
  R19 a sample path of length l ending at layer i is the tuple of the token's selected
      expert SETS (sorted ascending) at layers i-l+1 .. i (l >= 1 layers); estimation of
      layer m needs the m >= l layers before it ("starting from the l-th layer").
  R20 Ψ_j^{m}(e) = (tokens of group j that selected e in layer m) / (k · |group j|), a
      distribution over experts summing to 1.  A path never seen in profiling backs off to
      its suffixes of length l-1, ..., 1, then to layer m's marginal; a token with none of
      these contributes nothing.
  R21 top-k of Ψ by (count desc, expert id asc); P_j(e) = Ψ_j(e) for those k experts,
      0 otherwise; popularity(e) = (Σ_t P_{j(t)}(e) in token order) / N_t in fp64.
  R22 top-2k lists are compared as sets; ranking by (value desc, expert id asc) over
      all E experts (estimated popularity for phase one, actual selection counts for
      phase two).
Layers are 0-indexed here.
"""
from __future__ import annotations


def path_element(sel_t_layer) -> tuple:
    """The experts one token selected in one layer, as a sorted tuple (R19)."""
    return tuple(sorted(int(e) for e in sel_t_layer))


class Profile:
    """Per-layer sample-path counts: psi[(m, s, path)] = [count per expert] for the
    tokens whose last s layers before layer m match `path`, plus marg[m]."""

    def __init__(self, num_layers: int, num_experts: int, k: int, path_len: int):
        if path_len < 1:
            raise ValueError("path length l >= 1 (R19)")
        self.L, self.E, self.k, self.l = num_layers, num_experts, k, path_len
        self.psi: dict = {}
        self.marg: dict = {}

    def add_trace(self, sel):
        """'collect the expert selection results of all tokens': sel[t][i][:k]."""
        for t in range(len(sel)):
            elems = [path_element(sel[t][i]) for i in range(self.L)]
            for m in range(self.L):
                c = self.marg.setdefault(m, [0] * self.E)
                for e in elems[m]:
                    c[e] += 1
                for s in range(1, min(self.l, m) + 1):
                    key = (m, s, tuple(elems[m - s:m]))
                    c = self.psi.setdefault(key, [0] * self.E)
                    for e in elems[m]:
                        c[e] += 1

    def distribution(self, m: int, history) -> list | None:
        """Counts of Ψ for a token whose selections at layers m-l..m-1 are `history` (R20)."""
        elems = [path_element(h) for h in history]
        for s in range(self.l, 0, -1):
            key = (m, s, tuple(elems[len(elems) - s:]))
            if key in self.psi:
                return self.psi[key]
        return self.marg.get(m)


def top_k(counts, k: int) -> list:
    """The k experts with the largest counts, ties to the lower id (R21)."""
    return sorted(range(len(counts)), key=lambda e: (-counts[e], e))[:k]


def estimate(profile: Profile, m: int, histories):
    """Phase-one estimate of layer m's expert popularity for a batch.

    histories[t] = token t's selections at layers m-l .. m-1.  Returns (popularity[E],
    per-token top-k lists; [] for a token with no distribution)."""
    if m < profile.l:
        raise ValueError(f"layer {m} < path length {profile.l}: no sample path yet (R19)")
    E, k = profile.E, profile.k
    acc = [0.0] * E
    picks = []
    for hist in histories:
        c = profile.distribution(m, hist)
        if c is None or sum(c) == 0:
            picks.append([])
            continue
        total = sum(c)
        chosen = top_k(c, k)
        for e in chosen:
            acc[e] += c[e] / total            # P_j(e) = Ψ_j(e)
        picks.append(chosen)
    n_t = len(histories)
    return [a / n_t if n_t else 0.0 for a in acc], picks


def top2k_set(values, k: int) -> frozenset:
    """'the overall top-2k experts', ranked by (value desc, id asc) (R22)."""
    return frozenset(sorted(range(len(values)), key=lambda e: (-values[e], e))[:2 * k])


def phase_two(estimated_popularity, actual_counts, k: int) -> bool:
    """True when the estimated and actual top-2k lists are identical (no fine-tuning)."""
    return top2k_set(estimated_popularity, k) == top2k_set(actual_counts, k)
