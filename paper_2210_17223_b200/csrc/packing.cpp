// Expert packing (§8(f) row 3, A14/K13): the controller and the one-time parameter exchange.
//
// "Ideally, the FFN and all-to-all micro-ops should take a similar time so that both
// compute capacity and network bandwidth are fully utilized ... starting with one expert
// per device, it iteratively increases the number of experts per device in powers of two,
// until the FFN computation exceeds that of the all-to-all micro-op" (§4.2).  "We
// embed a packing controller in the MoE model and it runs a single thread.  Expert packing
// is dynamically adjusted after 10 training steps.  In the forward pass, the controller
// records the completion times of all-to-all and FFN micro-ops.  When FFN micro-ops are
// shorter than all-to-all, the controller starts to pack experts.  First, we initialize
// the new process groups.  Second, the controller inserts a one-time synchronous
// all-to-all to exchange expert parameters between packed devices" (§6.1); "Expert
// packing is launched at the 10-th step of each training task and is adjusted every four
// steps" (§7.1).
//
// B200 design: the controller is host state fed with device-timed micro-op durations
// (lina_profile: expert-GEMM phases and the all-to-all micro-ops of the variable layout);
// the decision must be identical on every rank, so callers pass rank-agreed values (the
// max over ranks).  The "new process group" is the group communicator the layer splits
// off on first use (layer.cpp group_comm); the packed layer itself is the variable layout
// with desc.pack = m.  The parameter exchange copies each newly hosted expert from a rank
// that hosts it under the old factor — peer memory over NVLink (copy engines), bracketed
// by two barriers, i.e. synchronous as in the paper.
#include <cstring>

#include "ce.h"
#include "internal.h"

struct lina_pack_ctl {
  int world = 1, pack = 1, start = 10, every = 4;
  int64_t steps = 0, since = 0;
  double ffn = 0.0, a2a = 0.0;
};

namespace lina {

// The doubling rule: pack more while the FFN micro-op is shorter than the all-to-all one
// and the next power of two still divides the world (at most every expert on every rank).
int pack_decide(int world, int pack, double ffn_ms, double a2a_ms) {
  const int next = 2 * pack;
  if (ffn_ms < a2a_ms && next <= world && world % next == 0) return next;
  return pack;
}

void pack_weights(lina_comm* cm, int E, int m0, int m1, size_t expert_bytes, const void* w_from, void* w_to,
                  cudaStream_t s) {
  const int P = cm->world, me = cm->rank;
  const int Elb = E / P, El0 = m0 * Elb, El1 = m1 * Elb;
  std::vector<char*> src(P, nullptr);
  if (P > 1) {
    comm_barrier(cm, s);  // every rank's w_from is complete
    src = cm->ce->peers(w_from, s);
  } else {
    src[0] = (char*)w_from;
  }
  for (int i = 0; i < El1; ++i) {
    const int e = (me / m1) * El1 + i;  // hosted expert i under the new factor
    const int g0 = e / El0;             // its group under the old factor
    const int r = (g0 == me / m0) ? me : g0 * m0 + me % m0;  // self, else the member with my residue
    LINA_CUDA_CHECK(cudaMemcpyAsync((char*)w_to + (size_t)i * expert_bytes,
                                    src[r] + (size_t)(e - g0 * El0) * expert_bytes, expert_bytes,
                                    cudaMemcpyDeviceToDevice, s));
  }
  if (P > 1) comm_barrier(cm, s);  // nobody changes w_from before every rank has copied
}

}  // namespace lina

using namespace lina;

extern "C" {

lina_status lina_pack_decide(int32_t world, int32_t pack, double ffn_ms, double a2a_ms, int32_t* pack_next) {
  if (world < 1 || pack < 1 || (pack & (pack - 1)) != 0 || world % pack != 0 || !pack_next ||
      !(ffn_ms >= 0.0) || !(a2a_ms >= 0.0)) {
    set_error("lina_pack_decide: need world >= 1, pack a power of two dividing world, times >= 0, pack_next");
    return LINA_ERR_INVALID_ARGUMENT;
  }
  *pack_next = pack_decide(world, pack, ffn_ms, a2a_ms);
  return LINA_OK;
}

lina_status lina_pack_ctl_create(int32_t world, int32_t start_step, int32_t every, lina_pack_ctl** out) {
  if (world < 1 || start_step < 1 || every < 1 || !out) {
    set_error("lina_pack_ctl_create: need world >= 1, start_step >= 1, every >= 1, out");
    return LINA_ERR_INVALID_ARGUMENT;
  }
  auto* c = new lina_pack_ctl();
  c->world = world;
  c->start = start_step;
  c->every = every;
  *out = c;
  return LINA_OK;
}

lina_status lina_pack_ctl_step(lina_pack_ctl* c, double ffn_ms, double a2a_ms, int32_t* pack, int32_t* changed) {
  if (!c || !pack || !(ffn_ms >= 0.0) || !(a2a_ms >= 0.0)) {
    set_error("lina_pack_ctl_step: NULL controller / pack, or a negative / NaN time");
    return LINA_ERR_INVALID_ARGUMENT;
  }
  ++c->steps;
  c->ffn += ffn_ms;
  c->a2a += a2a_ms;
  ++c->since;
  int ch = 0;
  // decide at step `start`, then every `every` steps, on the mean since the last decision
  if (c->steps >= c->start && (c->steps - c->start) % c->every == 0) {
    const int next = pack_decide(c->world, c->pack, c->ffn / c->since, c->a2a / c->since);
    ch = next != c->pack;
    c->pack = next;
    c->ffn = c->a2a = 0.0;
    c->since = 0;
  }
  *pack = c->pack;
  if (changed) *changed = ch;
  return LINA_OK;
}

lina_status lina_pack_ctl_destroy(lina_pack_ctl* c) {
  delete c;
  return LINA_OK;
}

}  // extern "C"
