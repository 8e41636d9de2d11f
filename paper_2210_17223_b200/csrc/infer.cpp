// S10: inference forward with popularity-driven expert replication.
//
// PAPER.md §5.2: replica counts n_e = N·Σ_t P(e)/N_t (Eq. 1), first-fit-
// decreasing packing; §6.2: the plan carries "how many tokens
// each replica should handle", the all-to-all uses an unequal split with no
// transfer to peers that get no tokens, hosted experts run on their device
// and the second all-to-all follows them.
//
// B200 design: every rank holds all E experts in HBM (the paper's
// host-DRAM copy, moved on-device), so a placement change moves no weights.
// The plan is computed identically on every rank from the allgathered per-source
// counts (no device-0 scheduler, no send/broadcast control plane); the default
// popularity is this batch's histogram (the paper's "w/o estimation" variant, P:905,
// reading R17).  One host synchronisation per call reads the counts (the unequal
// all-to-all needs host-visible sizes; H9).  Per call:
//   s : gate+softmax+top-k -> dropless slots (C = T) -> per-expert counts
//   s : allgather counts [P][E] -> D2H -> host plan (Eq. 1 + FFD, replica splits,
//       send/recv sizes) -> H2D of the routing tables
//   s : replica-routed permute -> one ncclSend/ncclRecv per peer (source-major
//       blocks) -> regroup expert-major (one padded segment per hosted expert) ->
//       grouped expert GEMMs over the hosted experts (tcgen05, weight index per
//       segment) -> regroup source-major -> one send/recv per peer back -> row-indexed
//       combine.
#include <algorithm>
#include <cstring>
#include <vector>

#include "ce.h"
#include "internal.h"
#include "kernels.h"
#include "layer.h"

namespace lina {

static size_t al(size_t x) { return (x + 255) / 256 * 256; }

struct InferPlan {
  int T, d, f, E, k, P, mpd, dt;
  size_t Cmax;
  size_t o_probs, o_idx, o_gate, o_slot, o_counts, o_kept, o_tokof, o_route, o_all, o_tab, o_vc,
      o_mtp, o_gvc, o_segx, o_blk, o_arow, o_send, o_recv, o_gin, o_h, o_o, o_back2, o_back, total;
  uint64_t peer_key;
  size_t tab_ints() const { return (size_t)E + (size_t)E * P + (size_t)P * E + E; }
};

static InferPlan infer_plan(const lina_moe_desc& dsc, int P, int mpd) {
  InferPlan q{};
  q.T = dsc.num_tokens;
  q.d = dsc.d_model;
  q.f = dsc.d_ffn;
  q.E = dsc.num_experts;
  q.k = dsc.k;
  q.P = P;
  q.mpd = mpd;
  q.dt = dsc.dtype == LINA_BF16 ? 2 : 4;
  const size_t Tk = (size_t)q.T * q.k;
  // expert-major segment pitch, worst case: every source's tokens to one expert
  q.Cmax = std::max<size_t>(128, ((size_t)P * Tk + 127) / 128 * 128);
  const size_t segs = (size_t)P * mpd;
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t at = o;
    o = al(o + b);
    return at;
  };
  // peer-written regions first (a rank stores into a peer's workspace at its own offsets)
  q.o_recv = take((size_t)P * Tk * q.d * q.dt);          // source-major receive       [peer-written]
  q.o_back = take(Tk * q.d * q.dt);                      // returned rows               [peer-written]
  q.o_probs = take(4 * (size_t)q.T * q.E);
  q.o_idx = take(4 * Tk);
  q.o_gate = take(4 * Tk);
  q.o_slot = take(4 * Tk);
  q.o_counts = take(4 * (size_t)q.E);
  q.o_kept = take(4 * (size_t)q.E);
  q.o_tokof = take(4 * (size_t)q.E * std::max(q.T, 1));
  q.o_route = take(4 * route_scratch_ints(q.T, q.k, q.E));
  q.o_all = take(4 * (size_t)P * q.E);
  q.o_tab = take(4 * q.tab_ints());
  q.o_vc = take(4 * segs);                 // rows received per (source, hosted expert)
  q.o_mtp = take(4 * ((size_t)mpd + 1));   // tile prefix over the hosted experts
  q.o_gvc = take(4 * (size_t)mpd);         // rows per hosted expert (all sources)
  q.o_segx = take(4 * (size_t)mpd);
  q.o_blk = take(4 * 6 * (size_t)P);        // fused exchange: {src_row, dst_row, rows} per peer, both ways
  q.o_arow = take(4 * Tk);
  q.o_send = take(Tk * q.d * q.dt);
  q.o_gin = take((size_t)mpd * q.Cmax * q.d * q.dt);     // expert-major GEMM input
  q.o_h = take((size_t)mpd * q.Cmax * q.f * q.dt);
  q.o_o = take((size_t)mpd * q.Cmax * q.d * q.dt);
  q.o_back2 = take((size_t)P * Tk * q.d * q.dt);         // outputs regrouped source-major
  q.total = o;
  uint64_t h = 1469598103934665603ull;  // FNV-1a of the peer-visible geometry
  for (uint64_t v : {(uint64_t)q.T, (uint64_t)q.k, (uint64_t)q.E, (uint64_t)q.d, (uint64_t)q.dt, (uint64_t)P,
                     (uint64_t)q.o_recv, (uint64_t)q.o_back, (uint64_t)0x1f})
    for (int b = 0; b < 8; ++b) h = (h ^ ((v >> (8 * b)) & 0xff)) * 1099511628211ull;
  q.peer_key = h | 1;
  return q;
}

size_t infer_workspace_bytes(const lina_moe_desc& desc, int world, int mpd) {
  return infer_plan(desc, world, std::max(1, mpd)).total;
}

static int* pinned(lina_comm* cm, size_t ints) {
  if (cm->pinned_bytes < ints * 4) {
    if (cm->pinned) cudaFreeHost(cm->pinned);
    cm->pinned = nullptr;
    cm->pinned_bytes = 0;
    LINA_CUDA_CHECK(cudaHostAlloc((void**)&cm->pinned, ints * 4, cudaHostAllocDefault));
    cm->pinned_bytes = ints * 4;
  }
  return cm->pinned;
}

void infer_forward(lina_comm* cm, const lina_moe_desc& desc, const void* tokens, const float* gate_w,
                   const void* w1_all, const void* w2_all, void* out, const lina_placement* placement,
                   int mpd_arg, lina_placement* plan_out, void* ws, size_t ws_bytes, cudaStream_t s,
                   const double* estimated, int32_t* replanned) {
  const int P = cm->world, rank = cm->rank;
  const int mpd = placement ? placement->max_per_device : mpd_arg;
  InferPlan q = infer_plan(desc, P, mpd);
  if (ws_bytes < q.total)
    throw StatusError{LINA_ERR_WORKSPACE, "workspace_bytes " + std::to_string(ws_bytes) + " < required " +
                                              std::to_string(q.total)};
  char* w = (char*)ws;
  float* probs = (float*)(w + q.o_probs);
  int* idx = (int*)(w + q.o_idx);
  float* gate = (float*)(w + q.o_gate);
  int* slot = (int*)(w + q.o_slot);
  int* counts = (int*)(w + q.o_counts);
  int* kept = (int*)(w + q.o_kept);
  int* tokof = (int*)(w + q.o_tokof);
  int* allc = (int*)(w + q.o_all);
  int* tab = (int*)(w + q.o_tab);
  int* vc = (int*)(w + q.o_vc);
  int* mtp = (int*)(w + q.o_mtp);
  int* gvc = (int*)(w + q.o_gvc);
  int* segx = (int*)(w + q.o_segx);
  int* blk = (int*)(w + q.o_blk);
  int* arow = (int*)(w + q.o_arow);
  char* send = w + q.o_send;
  char* recv = w + q.o_recv;
  char* gin = w + q.o_gin;
  char* hbuf = w + q.o_h;
  char* obuf = w + q.o_o;
  char* back2 = w + q.o_back2;
  char* back = w + q.o_back;
  const int T = q.T, E = q.E, k = q.k, d = q.d, f = q.f, dt = q.dt;
  const int dtype = desc.dtype == LINA_BF16 ? 1 : 0;
  const ncclDataType_t ndt = dtype ? ncclBfloat16 : ncclFloat32;

  trace_flush(cm);
  trace_mark(cm, s, "inf:start");
  // Fused exchange (peer stores, in-kernel flags) when the comm has the IPC transport;
  // NCCL send/recv otherwise.  This call's round is *round_inf + 1, closed at its end.
  CeTransport* ce = (P > 1 && cm->ce && cm->transport == 2) ? cm->ce : nullptr;
  uint32_t* ri = ce ? ce->round_inf() : nullptr;
  auto isig = [&](int wait_kind, int post_kind, int site, uint32_t* bump) {
    PeerSignal g;
    g.P = P;
    g.me = rank;
    g.stride = CeTransport::kMaxChunks;
    if (wait_kind >= 0) {
      g.wait = ce->slots(wait_kind);
      g.wait_round = ri;
      g.wait_add = 1;
    }
    if (post_kind >= 0) {
      g.post = ce->peer_slots(post_kind);
      g.post_round = ri;
      g.post_add = 1;
    }
    g.done = site >= 0 ? ce->done_counter(site) : nullptr;
    g.bump = bump;
    return g;
  };
  if (ce) {  // my receive and return buffers were last read by the previous call
    launch_sig_wait(isig(-1, CeTransport::kIFreeD, -1, nullptr), s);
    launch_sig_wait(isig(-1, CeTransport::kIFreeC, -1, nullptr), s);
  }
  // ---- gate, dropless slots, counts (S1, S2 with C = T)
  launch_gate_topk(dtype, tokens, gate_w, T, d, E, k, 1, probs, idx, gate, s);
  launch_route(idx, T, k, E, std::max(T, 1), (int*)(w + q.o_route), slot, counts, kept, tokof, s, cm->route_sync);
  const size_t ctrl_ints = (size_t)P * E + q.tab_ints() + (size_t)P * mpd + (mpd + 1) + 2 * (size_t)mpd + 6 * (size_t)P;
  int* host = pinned(cm, ctrl_ints);
  if (P > 1 && cm->host_allgather) {  // host-bootstrap communicator: counts through the host
    std::vector<int> mine((size_t)E);
    LINA_CUDA_CHECK(cudaMemcpyAsync(mine.data(), counts, 4 * (size_t)E, cudaMemcpyDeviceToHost, s));
    LINA_CUDA_CHECK(cudaStreamSynchronize(s));
    host_allgather(cm, mine.data(), host, 4 * (size_t)E);
    trace_mark(cm, s, "inf:gate+route+counts");
  } else {
    if (P > 1) {
      LINA_NCCL_CHECK(ncclAllGather(counts, allc, (size_t)E, ncclInt32, cm->ep_disp, s));
    } else {
      LINA_CUDA_CHECK(cudaMemcpyAsync(allc, counts, 4 * (size_t)E, cudaMemcpyDeviceToDevice, s));
    }
    trace_mark(cm, s, "inf:gate+route+counts");
    LINA_CUDA_CHECK(cudaMemcpyAsync(host, allc, 4 * (size_t)P * E, cudaMemcpyDeviceToHost, s));
    LINA_CUDA_CHECK(cudaStreamSynchronize(s));
  }
  std::vector<int> cnt(host, host + (size_t)P * E);  // cnt[src*E + e]
  {  // dropless: every source sends T·k rows; the receive regions are sized for equal T
    std::string bad;
    for (int src = 0; src < P; ++src) {
      long long tot = 0;
      for (int e = 0; e < E; ++e) tot += cnt[(size_t)src * E + e];
      if (tot != (long long)T * k) bad += " " + std::to_string(src);
    }
    if (!bad.empty())  // every rank sees the same counts: all of them raise
      throw ArgError{"inference needs num_tokens equal on every rank; rank(s)" + bad + " differ"};
  }

  // ---- the plan (identical on every rank).  Phase two: a phase-one plan
  // whose estimated top-2k experts differ from the actual ones is re-computed below.
  bool use_given = placement != nullptr;
  if (placement && estimated) {
    std::vector<int32_t> actual(E, 0);
    for (int src = 0; src < P; ++src)
      for (int e = 0; e < E; ++e) actual[e] += cnt[(size_t)src * E + e];
    use_given = phase_two_identical(estimated, actual.data(), E, k);
  }
  if (replanned) *replanned = (placement && !use_given) ? 1 : 0;
  std::vector<int> r(E), rdev((size_t)E * P, -1), hosted((size_t)P * mpd, -1);
  if (use_given) {
    const int mr = placement->max_replicas;
    for (int e = 0; e < E; ++e) {
      r[e] = placement->replicas[e];
      for (int i = 0; i < r[e]; ++i) rdev[(size_t)e * P + i] = placement->replica_device[(size_t)e * mr + i];
    }
    for (int dv = 0; dv < P; ++dv)
      for (int i = 0; i < mpd; ++i) hosted[(size_t)dv * mpd + i] = placement->hosted[(size_t)dv * mpd + i];
  } else {
    std::vector<double> pop(E, 0.0);
    double tot = 0.0;
    for (int src = 0; src < P; ++src)
      for (int e = 0; e < E; ++e) tot += cnt[(size_t)src * E + e];
    for (int e = 0; e < E; ++e) {
      double c = 0.0;
      for (int src = 0; src < P; ++src) c += cnt[(size_t)src * E + e];
      pop[e] = tot > 0 ? c / tot : 1.0 / E;
    }
    std::vector<int32_t> rr(E), rd((size_t)E * P), hs((size_t)P * mpd);
    lina_placement pl{E, P, mpd, P, rr.data(), rd.data(), hs.data()};
    std::string err;
    lina_status st = placement_compute(pop.data(), E, P, mpd, &pl, &err);
    if (st != LINA_OK) throw StatusError{st, err};
    for (int e = 0; e < E; ++e) {
      r[e] = rr[e];
      for (int i = 0; i < P; ++i) rdev[(size_t)e * P + i] = rd[(size_t)e * P + i];
    }
    hosted.assign(hs.begin(), hs.end());
  }
  // replica of e on device dv (-1 if none)
  auto replica_on = [&](int e, int dv) {
    for (int i = 0; i < r[e]; ++i)
      if (rdev[(size_t)e * P + i] == dv) return i;
    return -1;
  };
  std::vector<int> split(P);
  auto tokens_to = [&](int src, int e, int dv) {  // tokens src sends to dv for expert e (R14)
    const int i = replica_on(e, dv);
    if (i < 0) return 0;
    replica_split(cnt[(size_t)src * E + e], r[e], src, split.data());
    return split[i];
  };
  std::vector<int> nsend((size_t)P * E, 0), soff((size_t)P * E, 0), nrecv((size_t)P * mpd, 0);
  std::vector<int> dv_off(P, 0), dv_cnt(P, 0);  // this rank's block for each device (one message)
  int off = 0;
  for (int dv = 0; dv < P; ++dv) {
    dv_off[dv] = off;
    for (int i = 0; i < mpd; ++i) {
      const int e = hosted[(size_t)dv * mpd + i];
      if (e < 0) continue;
      soff[(size_t)dv * E + e] = off;
      nsend[(size_t)dv * E + e] = tokens_to(rank, e, dv);
      off += nsend[(size_t)dv * E + e];
    }
    dv_cnt[dv] = off - dv_off[dv];
  }
  std::vector<int> src_off(P, 0), src_cnt(P, 0), tot(mpd, 0);  // source-major receive blocks
  int roff = 0, maxseg = 0;
  for (int src = 0; src < P; ++src) {
    src_off[src] = roff;
    for (int h = 0; h < mpd; ++h) {
      const int e = hosted[(size_t)rank * mpd + h];
      const int n = e < 0 ? 0 : tokens_to(src, e, rank);
      nrecv[(size_t)src * mpd + h] = n;
      tot[h] += n;
      roff += n;
      maxseg = std::max(maxseg, n);
    }
    src_cnt[src] = roff - src_off[src];
  }
  // rows every source sends every device (identical on all ranks): where my blocks land
  std::vector<int> cnt_sd((size_t)P * P, 0);
  for (int src = 0; src < P; ++src)
    for (int dv = 0; dv < P; ++dv)
      for (int i = 0; i < mpd; ++i) {
        const int e = hosted[(size_t)dv * mpd + i];
        if (e >= 0) cnt_sd[(size_t)src * P + dv] += tokens_to(src, e, dv);
      }
  cm->inf_recv_rows.assign(src_cnt.begin(), src_cnt.end());
  cm->inf_sent_rows.assign(dv_cnt.begin(), dv_cnt.end());
  int maxrows = 0;
  for (int h = 0; h < mpd; ++h) maxrows = std::max(maxrows, tot[h]);
  const int Cm = std::max(128, (maxrows + 127) / 128 * 128);
  if ((size_t)Cm > q.Cmax) throw StatusError{LINA_ERR_WORKSPACE, "receive segment exceeds workspace"};

  // ---- routing tables to the device
  int* h = host;
  int* h_tab = h;
  for (int e = 0; e < E; ++e) h_tab[e] = r[e];
  for (size_t i = 0; i < (size_t)E * P; ++i) h_tab[E + i] = rdev[i];
  for (size_t i = 0; i < (size_t)P * E; ++i) h_tab[E + (size_t)E * P + i] = soff[i];
  for (int e = 0; e < E; ++e) h_tab[E + 2 * (size_t)E * P + e] = cnt[(size_t)rank * E + e];
  int* h_vc = h_tab + q.tab_ints();
  int* h_mtp = h_vc + (size_t)P * mpd;
  int* h_gvc = h_mtp + (mpd + 1);
  int* h_segx = h_gvc + mpd;
  const int rows = tc_tile_rows();
  for (int i = 0; i < P * mpd; ++i) h_vc[i] = nrecv[i];
  int run = 0;
  for (int i = 0; i < mpd; ++i) {
    h_gvc[i] = tot[i];
    h_mtp[i] = run;
    run += (tot[i] + rows - 1) / rows;
  }
  h_mtp[mpd] = run;
  for (int i = 0; i < mpd; ++i) h_segx[i] = std::max(0, hosted[(size_t)rank * mpd + i]);
  int* h_blk = h_segx + mpd;
  int maxblk = 0;
  for (int o = 0; o < P; ++o) {
    int at_o = 0, at_me = 0;  // my block's row in o's receive buffer / o's block's row in my return buffer
    for (int s2 = 0; s2 < rank; ++s2) at_o += cnt_sd[(size_t)s2 * P + o];
    for (int dv = 0; dv < rank; ++dv) at_me += cnt_sd[(size_t)o * P + dv];
    h_blk[3 * o] = dv_off[o];  // dispatch: my send block for device o -> o's receive (source-major)
    h_blk[3 * o + 1] = at_o;
    h_blk[3 * o + 2] = dv_cnt[o];
    h_blk[3 * (P + o)] = src_off[o];  // return: rows source o sent me -> o's return buffer
    h_blk[3 * (P + o) + 1] = at_me;
    h_blk[3 * (P + o) + 2] = src_cnt[o];
    maxblk = std::max(maxblk, std::max(dv_cnt[o], src_cnt[o]));
  }
  LINA_CUDA_CHECK(cudaMemcpyAsync(tab, h_tab, 4 * q.tab_ints(), cudaMemcpyHostToDevice, s));
  LINA_CUDA_CHECK(cudaMemcpyAsync(vc, h_vc, 4 * (size_t)P * mpd, cudaMemcpyHostToDevice, s));
  LINA_CUDA_CHECK(cudaMemcpyAsync(mtp, h_mtp, 4 * (size_t)(mpd + 1), cudaMemcpyHostToDevice, s));
  LINA_CUDA_CHECK(cudaMemcpyAsync(gvc, h_gvc, 4 * (size_t)mpd, cudaMemcpyHostToDevice, s));
  LINA_CUDA_CHECK(cudaMemcpyAsync(segx, h_segx, 4 * (size_t)mpd, cudaMemcpyHostToDevice, s));
  if (ce) LINA_CUDA_CHECK(cudaMemcpyAsync(blk, h_blk, 4 * 6 * (size_t)P, cudaMemcpyHostToDevice, s));

  trace_mark(cm, s, "inf:plan+tables(host)");
  // ---- replica-routed permute and the unequal-split all-to-all
  launch_infer_permute(dtype, tokens, idx, slot, tab, T, k, d, E, P, rank, send, arow, s);
  trace_mark(cm, s, "inf:permute");
  // one message per peer: my block for device dv -> its source-major receive block
  if (ce) {  // peer stores (after the owners' FREE; READY when every block has landed)
    void* const* peer_recv = ce->dev_ptrs(ws, q.o_recv, s, q.peer_key);
    launch_sig_wait(isig(CeTransport::kIFreeD, -1, -1, nullptr), s);
    launch_push_blocks(dtype, send, peer_recv, blk, P, d, maxblk, isig(-1, CeTransport::kIReadyD, 6, nullptr), s);
    launch_sig_wait(isig(CeTransport::kIReadyD, -1, -1, nullptr), s);
  } else if (P > 1) {
    LINA_NCCL_CHECK(ncclGroupStart());
    for (int dv = 0; dv < P; ++dv)
      if (dv_cnt[dv])
        LINA_NCCL_CHECK(ncclSend(send + (size_t)dv_off[dv] * d * dt, (size_t)dv_cnt[dv] * d, ndt, dv, cm->ep_disp, s));
    for (int src = 0; src < P; ++src)
      if (src_cnt[src])
        LINA_NCCL_CHECK(ncclRecv(recv + (size_t)src_off[src] * d * dt, (size_t)src_cnt[src] * d, ndt, src,
                                 cm->ep_disp, s));
    LINA_NCCL_CHECK(ncclGroupEnd());
  } else if (dv_cnt[0]) {
    LINA_CUDA_CHECK(cudaMemcpyAsync(recv, send, (size_t)dv_cnt[0] * d * dt, cudaMemcpyDeviceToDevice, s));
  }
  launch_regroup(dtype, recv, gin, vc, P, mpd, Cm, d, maxseg, true, s);
  trace_mark(cm, s, "inf:a2av dispatch");
  // ---- expert FFN over the hosted experts (S5; one launch per GEMM for every segment)
  RowGemm g1{};
  g1.A = gin;
  g1.B = w1_all;
  g1.D = hbuf;
  g1.vcount = gvc;
  g1.mtp = mtp;
  g1.seg0 = 0;
  g1.nseg = mpd;
  g1.El = mpd;
  g1.Cm = Cm;
  g1.N = f;
  g1.K = d;
  g1.seg_expert = segx;
  g1.B_experts = E;
  RowGemm g2 = g1;
  g2.A = hbuf;
  g2.B = w2_all;
  g2.D = obuf;
  g2.N = d;
  g2.K = f;
  prof_begin(cm, s);
  launch_expert_row_gemm(dtype, g1, true, kEpiRelu, s);
  launch_expert_row_gemm(dtype, g2, true, kEpiNone, s);
  prof_end(cm, s, 2);
  trace_mark(cm, s, "inf:expert GEMMs");

  // ---- second all-to-all (expert outputs back to their sources, one message per peer)
  launch_regroup(dtype, obuf, back2, vc, P, mpd, Cm, d, maxseg, false, s);
  if (ce) {  // the rows go back by peer stores; the last wait also closes this call's round
    void* const* peer_back = ce->dev_ptrs(ws, q.o_back, s, q.peer_key);
    launch_sig_wait(isig(CeTransport::kIFreeC, -1, -1, nullptr), s);
    launch_push_blocks(dtype, back2, peer_back, blk + 3 * P, P, d, maxblk, isig(-1, CeTransport::kIReadyC, 7, nullptr),
                       s);
    launch_sig_wait(isig(CeTransport::kIReadyC, -1, -1, ri), s);
  } else if (P > 1) {
    LINA_NCCL_CHECK(ncclGroupStart());
    for (int src = 0; src < P; ++src)
      if (src_cnt[src])
        LINA_NCCL_CHECK(ncclSend(back2 + (size_t)src_off[src] * d * dt, (size_t)src_cnt[src] * d, ndt, src,
                                 cm->ep_comb, s));
    for (int dv = 0; dv < P; ++dv)
      if (dv_cnt[dv])
        LINA_NCCL_CHECK(ncclRecv(back + (size_t)dv_off[dv] * d * dt, (size_t)dv_cnt[dv] * d, ndt, dv, cm->ep_comb, s));
    LINA_NCCL_CHECK(ncclGroupEnd());
  } else if (dv_cnt[0]) {
    LINA_CUDA_CHECK(cudaMemcpyAsync(back, back2, (size_t)dv_cnt[0] * d * dt, cudaMemcpyDeviceToDevice, s));
  }
  trace_mark(cm, s, "inf:a2av combine");
  launch_combine_rows(dtype, back, arow, gate, T, k, d, out, s);
  trace_mark(cm, s, "inf:combine");

  if (plan_out) {
    plan_out->num_experts = E;
    plan_out->num_devices = P;
    plan_out->max_per_device = mpd;
    for (int e = 0; e < E; ++e) {
      plan_out->replicas[e] = r[e];
      for (int i = 0; i < plan_out->max_replicas; ++i)
        plan_out->replica_device[(size_t)e * plan_out->max_replicas + i] = i < P ? rdev[(size_t)e * P + i] : -1;
    }
    for (size_t i = 0; i < (size_t)P * mpd; ++i) plan_out->hosted[i] = hosted[i];
  }
}

}  // namespace lina
