// The MoE layer pipeline: forward (S1-S7) and backward (S8) with the Lina
// micro-op pipelining of the all-to-all against the expert GEMMs.
//
// Forward, per rank ("the expert can start computing with a
// subset of the tokens after one all-to-all micro-op"; "FFN is ready to
// start right after each all-to-all micro-op"):
//   s  : gate+softmax+top-k -> route (slot, tok_of) -> permute into Send[n][E][Cm][d]
//   hi : count all-to-all (kept[E] -> recv_kept[P][E_l])
//   for c: hi : all-to-all Send[c] -> Recv[c]                     (dispatch micro-op)
//   for c: s  : wait dispatch c; GEMM1+ReLU, GEMM2 on Recv[c]      (expert micro-op)
//   for c: hi2: wait GEMM c; all-to-all Out[c] -> Back[c]          (combine micro-op)
//   s  : wait combine n-1; weighted un-permute -> y
// Host enqueue order is all dispatches, then GEMMs, then combines (H8 in
// SURVEY.md): NCCL runs one communicator's operations in issue order, so an
// interleaved order would make dispatch c+1 wait behind combine c.  Dispatch and
// combine use separate communicators/streams so both link directions overlap.
// The host only enqueues: no host<->device synchronisation anywhere, so the
// whole sequence is CUDA-graph capturable.  At P = 1 there is no collective and
// Recv/Back alias Send/Out.
#include <cstring>

#include "internal.h"
#include "kernels.h"
#include "ce.h"
#include "layer.h"

namespace lina {

static size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

Plan make_plan(const lina_moe_desc& dsc, int world) {
  Plan p{};
  p.T = dsc.num_tokens;
  p.d = dsc.d_model;
  p.f = dsc.d_ffn;
  p.E = dsc.num_experts;
  p.k = dsc.k;
  p.C = dsc.capacity;
  p.n = dsc.n_chunks;
  p.P = world;
  p.El = dsc.num_experts / world;
  p.Cm = chunk_rows_max(p.C, p.n);
  p.bf16 = dsc.dtype == LINA_BF16;
  p.dt = p.bf16 ? 2 : 4;
  // M tile of the expert row GEMMs: 256-row CTA pairs (the pair splits the weight tile, so
  // each weight slab is read once per segment up to 256 rows) unless a segment (one source's
  // rows of one expert) averages <= 96 rows, where 128-row tiles halve the idle MMA rows and
  // a segment still mostly fits one tile.  At ~128 rows (C4) the pairs measured 2% faster
  // (profiles/r01_bench_c4_n1.json).  LINA_TILE_ROWS=128|256 overrides.
  {
    const long long per_seg = (long long)p.T * p.k / std::max(1, p.E);
    p.tile_rows = per_seg <= 96 ? 128 : 256;
    const char* tr = getenv("LINA_TILE_ROWS");
    if (tr && (atoi(tr) == 128 || atoi(tr) == 256)) p.tile_rows = atoi(tr);
    // tail split of the 256-row tiles (RowGemm::mtp_tail): tensor-core path only, opt-in
    // (LINA_TAIL128=1).  Its second launch has one 128-row tile per segment and N block, each
    // with the full K: at C2 / C3 that is less than a wave of long tiles, which cost more
    // than the halved padding saves (C2 N=1: 0.512 vs 0.443 ms per step; C3 N=2: 0.945 vs
    // 0.890 ms); at C5 the two roughly cancel (profiles/r02_tail_split_ab.txt).
    const char* ts = getenv("LINA_TAIL128");
    p.tail_split = p.bf16 && p.tile_rows == 256 && (ts && ts[0] == '1') && !getenv("LINA_FORCE_SIMT");
    // half tails: the same saving without the second launch — a segment's last <= 128 rows
    // as an M = 128 cta_group::2 tile inside the 256-row launch (gemm_tc.cu); LINA_HALF128=0|1
    const char* ht = getenv("LINA_HALF128");
    p.half_tails = p.bf16 && p.tile_rows == 256 && !p.tail_split && !(ht && ht[0] == '0') &&
                   !getenv("LINA_FORCE_SIMT");
  }
  const size_t T = p.T, k = p.k, E = p.E;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = align_up(o + bytes);
    return at;
  };
  const int pack = dsc.pack > 1 ? dsc.pack : 1;
  if (dsc.capacity == 0 || pack > 1) {
    // variable layout: dropless (capacity 0, §8(f) row 4: count exchange + unequal split)
    // and/or expert packing (pack > 1: m·E_l experts per rank, groups of m ranks)
    p.dropless = true;
    p.pack = pack;
    p.El = pack * p.E / p.P;  // experts hosted per rank
    p.C = dsc.capacity > 0 ? dsc.capacity : std::max(p.T, 1);  // capacity 0: slots never run out
    p.n = 1;
    const int R = p.tile_rows;
    p.Cm = R;
    // virtual segments: Σ_{(el, source)} ceil(c / R) <= rows / R + (P/m)·m·E_l, with the
    // P/m sources of a rank sending it rows <= (P/m)·T·min(k, hosted experts)
    const long long rows =
        (long long)(p.P / pack) * std::min((long long)p.T * std::min(p.k, p.El), (long long)p.C * p.El);
    p.V = (int)(rows / R + (long long)p.E + 1);
    const size_t vrows = (size_t)p.V * R, srows = (size_t)p.T * p.k;
    const size_t tab_ints = 2 * E + (size_t)p.P * E + p.P + 4 * (size_t)p.V + 2 * (size_t)(p.V + 1) + 2 * (size_t)p.El;
    // peer-visible regions first (T-independent offsets are not possible here: the
    // source-compact buffers hold T·k rows, so dropless needs equal T on every rank)
    p.s_R = take(vrows * p.d * p.dt);                                    // [peer-written]
    p.s_C = take((p.P > 1 ? srows : vrows) * p.d * p.dt);                // [peer-written] (P=1: O itself)
    p.s_allc = take(4 * (size_t)p.P * E);                                // [peer-written]
    p.s_kept = take(4 * E);
    p.s_probs = take(4 * T * E);
    p.s_idx = take(4 * T * k);
    p.s_gate = take(4 * T * k);
    p.s_slot = take(4 * T * k);
    p.s_tokof = take(4 * E * (size_t)p.C);
    p.s_tab = take(4 * tab_ints);
    p.s_H = take(vrows * (size_t)p.f * p.dt);
    p.s_mask = take(vrows * (size_t)((p.f + 63) / 64) * 8);
    p.saved_bytes = o;
    o = 0;
    p.w_dO = take(vrows * p.d * p.dt);                                   // [peer-written]
    p.w_dXs = (p.P > 1) ? take(srows * p.d * p.dt) : 0;                  // [peer-written]
    p.w_O = (p.P > 1) ? take(vrows * p.d * p.dt) : 0;
    p.w_dXe = take(vrows * p.d * p.dt);
    p.w_route = take(4 * route_scratch_ints(p.T, p.k, p.E));
    p.w_dg = take(4 * T * k);
    p.w_dwg = take(4 * dwg_scratch_floats(p.T, p.d, p.E));
    p.w_dH = take(vrows * (size_t)p.f * p.dt);
    p.ws_bytes = o;
    uint64_t h = 1469598103934665603ull;
    for (uint64_t v : {(uint64_t)0xd1, (uint64_t)p.T, (uint64_t)p.k, (uint64_t)p.V, (uint64_t)R, (uint64_t)p.E,
                       (uint64_t)p.pack, (uint64_t)p.C,
                       (uint64_t)p.P, (uint64_t)p.d, (uint64_t)p.f, (uint64_t)p.dt, (uint64_t)p.s_R, (uint64_t)p.s_C,
                       (uint64_t)p.s_allc, (uint64_t)p.w_dO, (uint64_t)p.w_dXs})
      for (int b = 0; b < 8; ++b) h = (h ^ ((v >> (8 * b)) & 0xff)) * 1099511628211ull;
    p.peer_key = h | 1;
    return p;
  }
  const size_t send_rows = p.rows_send(), recv_rows = p.rows_recv();
  // Every region a peer writes or reads at this rank's offsets (fused / copy-engine
  // transports: a rank finds a peer's buffer as the peer's base + ITS OWN offset) comes
  // first, sized by (C, n_chunks, E, d, dtype, world) only, so ranks may pass different
  // num_tokens; the peer mapping checks every rank's peer_key (ce.cpp) on first use.
  // ---- saved (forward -> backward)
  p.s_R = take(recv_rows * p.d * p.dt);                       // routed tokens (X rows)     [peer-written]
  p.s_C = take(send_rows * p.d * p.dt);                       // returned expert outputs    [peer-written]
  p.s_recvkept = take(4 * (size_t)p.P * p.El);                // kept counts of each source [peer-written]
  p.s_kept = take(4 * E);                                     //                            [peer-read, ce]
  p.s_probs = take(4 * T * E);
  p.s_idx = take(4 * T * k);
  p.s_gate = take(4 * T * k);
  p.s_slot = take(4 * T * k);
  p.s_tokof = take(4 * E * (size_t)p.C);
  p.s_vcount = take(4 * (size_t)p.n * p.P * p.El);
  p.s_mtp = take(4 * (size_t)p.n * (p.P * p.El + 1));
  p.s_mtpt = take(4 * (size_t)p.n * (p.P * p.El + 1));
  p.s_rbase = take(4 * (size_t)p.n * p.P * p.El);
  p.s_H = take(recv_rows * (size_t)p.f * p.dt);               // relu(X W1ᵀ)
  p.s_mask = take(recv_rows * (size_t)((p.f + 63) / 64) * 8);  // ReLU' bits of H
  p.saved_bytes = o;
  // ---- workspace
  o = 0;
  p.w_dO = (p.P > 1) ? take(recv_rows * p.d * p.dt) : 0;      // (P=1: = dS)                [peer-written]
  p.w_dXs = (p.P > 1) ? take(send_rows * p.d * p.dt) : 0;     // (P=1: = dXe)               [peer-written]
  p.w_D = (p.P > 1) ? take(send_rows * p.d * p.dt) : 0;       // send buffer (P=1: = R)     [peer-read, ce]
  p.w_O = (p.P > 1) ? take(recv_rows * p.d * p.dt) : 0;       // expert outputs (P=1: = C)  [peer-read, ce]
  p.w_dS = take(send_rows * p.d * p.dt);                      // g·dY rows, send layout     [peer-read, ce]
  p.w_dXe = take(recv_rows * p.d * p.dt);                     //                            [peer-read, ce]
  p.w_route = take(4 * route_scratch_ints(p.T, p.k, p.E));
  p.w_dg = take(4 * T * k);
  p.w_dwg = take(4 * dwg_scratch_floats(p.T, p.d, p.E));
  p.w_dH = take(recv_rows * (size_t)p.f * p.dt);
  p.ws_bytes = o;
  // FNV-1a over the peer-visible geometry (equal on every rank or the mapping fails)
  uint64_t h = 1469598103934665603ull;
  for (uint64_t v : {(uint64_t)p.C, (uint64_t)p.n, (uint64_t)p.Cm, (uint64_t)p.E, (uint64_t)p.P, (uint64_t)p.d,
                     (uint64_t)p.f, (uint64_t)p.dt, (uint64_t)p.s_R, (uint64_t)p.s_C, (uint64_t)p.s_recvkept,
                     (uint64_t)p.s_kept, (uint64_t)p.w_dO, (uint64_t)p.w_dXs, (uint64_t)p.w_D, (uint64_t)p.w_O,
                     (uint64_t)p.w_dS, (uint64_t)p.w_dXe})
    for (int b = 0; b < 8; ++b) h = (h ^ ((v >> (8 * b)) & 0xff)) * 1099511628211ull;
  p.peer_key = h | 1;
  return p;
}

namespace {

struct Ptrs {
  float* probs; int* idx; float* gate; int* slot; int* kept; int* tok_of; int* recv_kept;
  int* vcount; int* mtp; int* mtpt; int* rbase; char* R; char* H; char* Cb; uint64_t* mask;
  int* route; char* D; char* O; float* dg; float* dwg; char* dS; char* dO; char* dH;
  char* dXe; char* dXs;
  int* allc;    // dropless: [P][E] exchanged counts
  DlTables dl;  // dropless: layout tables
};

Ptrs carve_dropless(const Plan& p, void* saved, void* ws) {
  char* sv = (char*)saved;
  char* w = (char*)ws;
  Ptrs q{};
  if (sv) {
    q.probs = (float*)(sv + p.s_probs);
    q.idx = (int*)(sv + p.s_idx);
    q.gate = (float*)(sv + p.s_gate);
    q.slot = (int*)(sv + p.s_slot);
    q.kept = (int*)(sv + p.s_kept);
    q.tok_of = (int*)(sv + p.s_tokof);
    q.allc = (int*)(sv + p.s_allc);
    q.R = sv + p.s_R;
    q.H = sv + p.s_H;
    q.Cb = sv + p.s_C;
    q.mask = (uint64_t*)(sv + p.s_mask);
    int* t = (int*)(sv + p.s_tab);
    const int E = p.E, P = p.P, V = p.V;
    q.dl.dbase = t;
    q.dl.ebase = t + E;
    q.dl.soff = t + 2 * E;
    q.dl.src_total = q.dl.soff + (size_t)P * E;
    q.dl.vcount = q.dl.src_total + P;
    q.dl.vexp = q.dl.vcount + V;
    q.dl.vsrc = q.dl.vexp + V;
    q.dl.vq0 = q.dl.vsrc + V;
    q.dl.mtp = q.dl.vq0 + V;
    q.dl.mtpt = q.dl.mtp + V + 1;
    q.dl.vrange = q.dl.mtpt + V + 1;
    q.vcount = q.dl.vcount;
    q.mtp = q.dl.mtp;
  }
  if (w) {
    q.route = (int*)(w + p.w_route);
    q.O = p.P > 1 ? w + p.w_O : q.Cb;  // P = 1: the expert outputs stay in `saved` (read back by backward)
    q.dg = (float*)(w + p.w_dg);
    q.dwg = (float*)(w + p.w_dwg);
    q.dO = w + p.w_dO;
    q.dH = w + p.w_dH;
    q.dXe = w + p.w_dXe;
    q.dXs = p.P > 1 ? w + p.w_dXs : q.dXe;
  }
  return q;
}

Ptrs carve(const Plan& p, void* saved, void* ws) {
  if (p.dropless) return carve_dropless(p, saved, ws);
  char* sv = (char*)saved;
  char* w = (char*)ws;
  Ptrs q{};
  if (sv) {
    q.probs = (float*)(sv + p.s_probs);
    q.idx = (int*)(sv + p.s_idx);
    q.gate = (float*)(sv + p.s_gate);
    q.slot = (int*)(sv + p.s_slot);
    q.kept = (int*)(sv + p.s_kept);
    q.tok_of = (int*)(sv + p.s_tokof);
    q.recv_kept = (int*)(sv + p.s_recvkept);
    q.vcount = (int*)(sv + p.s_vcount);
    q.mtp = (int*)(sv + p.s_mtp);
    q.mtpt = (int*)(sv + p.s_mtpt);
    q.rbase = (int*)(sv + p.s_rbase);
    q.R = sv + p.s_R;
    q.H = sv + p.s_H;
    q.Cb = sv + p.s_C;
    q.mask = (uint64_t*)(sv + p.s_mask);
  }
  if (w) {
    q.route = (int*)(w + p.w_route);
    q.D = p.P > 1 ? w + p.w_D : q.R;
    q.O = p.P > 1 ? w + p.w_O : q.Cb;
    q.dg = (float*)(w + p.w_dg);
    q.dwg = (float*)(w + p.w_dwg);
    q.dS = w + p.w_dS;
    q.dO = p.P > 1 ? w + p.w_dO : q.dS;
    q.dH = w + p.w_dH;
    q.dXe = w + p.w_dXe;
    q.dXs = p.P > 1 ? w + p.w_dXs : q.dXe;
  }
  return q;
}

ncclDataType_t nccl_dt(const Plan& p) { return p.bf16 ? ncclBfloat16 : ncclFloat32; }

// Equal-split all-to-all of chunk c of a send-layout buffer ([n][E][Cm][w]) into a
// receive-layout buffer ([n][P][E_l][Cm][w]).  Per peer: E_l*Cm*w elements.
void a2a_send_to_recv(const Plan& p, const char* send, char* recv, int w, int c, ncclComm_t comm,
                      cudaStream_t st) {
  const size_t per_peer = (size_t)p.El * p.Cm * w;
  const size_t chunk = per_peer * p.P;  // = E*Cm*w = P*El*Cm*w
  LINA_NCCL_CHECK(ncclAlltoAll(send + c * chunk * p.dt, recv + c * chunk * p.dt, per_peer,
                               nccl_dt(p), comm, st));
}
// Reverse: receive layout chunk c -> send layout chunk c (same sizes).
void a2a_recv_to_send(const Plan& p, const char* recv, char* send, int w, int c, ncclComm_t comm,
                      cudaStream_t st) {
  a2a_send_to_recv(p, recv, send, w, c, comm, st);
}

// The tail-split tile lists of chunk c (laid out after the main prefix in `saved`: mtp,
// then mtp_tail [n][nseg+1], then row_base [n][nseg]).
void set_tail(const Plan& p, RowGemm& g, const int* mtp, int c) {
  if (!p.tail_split || p.dropless) return;
  const size_t nseg = (size_t)p.P * p.El;
  g.mtp_tail = mtp + (p.s_mtpt - p.s_mtp) / 4 + (size_t)c * (nseg + 1);
  g.row_base = mtp + (p.s_rbase - p.s_mtp) / 4;  // [n][nseg]: indexed by the global segment
}
// After vcount (and the plain prefix) of every chunk: the tail-split lists.
void tile_lists(const Plan& p, const Ptrs& q, cudaStream_t s) {
  if (p.tail_split && !p.dropless) launch_mtile_split(q.vcount, p.n, p.P * p.El, q.mtp, q.mtpt, q.rbase, s);
}

void row_gemm(const Plan& p, const void* A, const void* B, void* D, const void* aux,
              const int* vcount, const int* mtp, int c, int N, int K, bool b_kmajor, int epi,
              cudaStream_t st, uint64_t* mask_out = nullptr, const uint64_t* mask_in = nullptr,
              const PeerSignal* sig = nullptr, int src_me = -1) {
  RowGemm g{};
  if (src_me >= 0) {  // split dispatch: sig.wait per source, tiles from source src_me up
    g.src_wait = 1;
    g.src_P = p.P;
    g.src_me = src_me;
  }
  g.tile_rows = p.tile_rows;
  g.half_tails = p.half_tails;
  g.sig = sig;
  g.mask_out = mask_out;
  g.mask_in = mask_in;
  g.mtp = mtp + (size_t)c * (p.P * p.El + 1);
  g.A = A;
  g.B = B;
  g.D = D;
  g.aux = aux;
  g.vcount = vcount;
  g.seg0 = c * p.P * p.El;
  g.nseg = p.P * p.El;
  g.El = p.El;
  g.Cm = p.Cm;
  g.N = N;
  g.K = K;
  set_tail(p, g, mtp, c);
  launch_expert_row_gemm(p.bf16 ? 1 : 0, g, b_kmajor, epi, st);
}

// ------------------------------------------------------------------ copy-engine transport
// (ce.cpp).  Byte offsets of the chunk blocks:
//   send layout [n][E][Cm][w]:        block of peer r in chunk c  = (c*E + r*El)*Cm*w
//   recv layout [n][P][El][Cm][w]:    segment of source s in chunk c = (c*P + s)*El*Cm*w
size_t send_block(const Plan& p, int c, int r, int w) { return ((size_t)c * p.E + (size_t)r * p.El) * p.Cm * w * p.dt; }
size_t recv_block(const Plan& p, int c, int s, int w) { return ((size_t)c * p.P + s) * p.El * p.Cm * w * p.dt; }
size_t block_bytes(const Plan& p, int w) { return (size_t)p.El * p.Cm * w * p.dt; }

// Forward micro-ops on the copy engines: dispatch pulls (peer D -> my R) per (source,
// chunk) on per-source streams, GEMMs per chunk as soon as every source's chunk is in,
// combine pulls (peer O -> my Cb) per chunk as soon as the expert rank posts it.
void forward_ce(lina_comm* cm, const Plan& p, const Ptrs& q, const void* w1, const void* w2,
                void* saved, void* ws, cudaEvent_t e_perm, uint32_t seq, bool compute, cudaStream_t s) {
  CeTransport& ce = *cm->ce;
  const int P = p.P, me = cm->rank, n = p.n, d = p.d;
  const auto& peer_ws = ce.peers(ws, s, p.peer_key);
  const auto& peer_saved = ce.peers(saved, s, p.peer_key);
  for (int src = 0; src < P; ++src) {
    cudaStream_t st = ce.disp_stream(src);
    LINA_CUDA_CHECK(cudaStreamWaitEvent(st, e_perm, 0));
    if (src != me) ce.wait_flag(st, CeTransport::kReadyFwdD, src, 0, seq);
    LINA_CUDA_CHECK(cudaMemcpyAsync(q.recv_kept + (size_t)src * p.El,
                                    peer_saved[src] + p.s_kept + 4 * (size_t)me * p.El, 4 * (size_t)p.El,
                                    cudaMemcpyDeviceToDevice, st));
    LINA_CUDA_CHECK(cudaEventRecord(ce.ev(0, src, CeTransport::kMaxChunks), st));
    for (int c = 0; c < n; ++c) {
      LINA_CUDA_CHECK(cudaMemcpyAsync(q.R + recv_block(p, c, src, d), peer_ws[src] + p.w_D + send_block(p, c, me, d),
                                      block_bytes(p, d), cudaMemcpyDeviceToDevice, st));
      LINA_CUDA_CHECK(cudaEventRecord(ce.ev(0, src, c), st));
    }
    if (src != me) ce.post_flag(st, src, CeTransport::kPulledFwdD, me, 0, seq);
  }
  for (int src = 0; src < P; ++src)
    LINA_CUDA_CHECK(cudaStreamWaitEvent(s, ce.ev(0, src, CeTransport::kMaxChunks), 0));
  if (compute) {
    launch_vcount(q.recv_kept, P, p.El, p.C, n, q.vcount, s);
    launch_mtile_prefix(q.vcount, n, P * p.El, p.tile_rows, q.mtp, s);
    tile_lists(p, q, s);
  }
  for (int r = 0; r < P; ++r)  // every peer has pulled my previous O
    if (r != me) ce.wait_flag(s, CeTransport::kPulledFwdC, r, 0, ce.prev_ce_fwd);
  for (int c = 0; c < n; ++c) {
    for (int src = 0; src < P; ++src) LINA_CUDA_CHECK(cudaStreamWaitEvent(s, ce.ev(0, src, c), 0));
    if (compute) {
      prof_begin(cm, s);
      row_gemm(p, q.R, w1, q.H, nullptr, q.vcount, q.mtp, c, p.f, p.d, true, kEpiRelu, s, q.mask);
      row_gemm(p, q.H, w2, q.O, nullptr, q.vcount, q.mtp, c, p.d, p.f, true, kEpiNone, s);
      prof_end(cm, s, 2);
    }
    for (int r = 0; r < P; ++r)
      if (r != me) ce.post_flag(s, r, CeTransport::kReadyFwdC, me, c, seq);
    LINA_CUDA_CHECK(cudaEventRecord(ce.ev(1, me, c), s));
  }
  for (int src = 0; src < P; ++src) {
    cudaStream_t st = ce.comb_stream(src);
    LINA_CUDA_CHECK(cudaStreamWaitEvent(st, e_perm, 0));
    for (int c = 0; c < n; ++c) {
      if (src == me) LINA_CUDA_CHECK(cudaStreamWaitEvent(st, ce.ev(1, me, c), 0));
      else ce.wait_flag(st, CeTransport::kReadyFwdC, src, c, seq);
      LINA_CUDA_CHECK(cudaMemcpyAsync(q.Cb + send_block(p, c, src, d), peer_ws[src] + p.w_O + recv_block(p, c, me, d),
                                      block_bytes(p, d), cudaMemcpyDeviceToDevice, st));
    }
    if (src != me) ce.post_flag(st, src, CeTransport::kPulledFwdC, me, 0, seq);
    LINA_CUDA_CHECK(cudaEventRecord(ce.ev(2, src, CeTransport::kMaxChunks), st));
  }
  for (int src = 0; src < P; ++src)
    LINA_CUDA_CHECK(cudaStreamWaitEvent(s, ce.ev(2, src, CeTransport::kMaxChunks), 0));
}

void backward_ce(lina_comm* cm, const Plan& p, const Ptrs& q, const void* w1, const void* w2, void* dw1,
                 void* dw2, void* ws, cudaEvent_t e_cb, uint32_t seq, int dtype, bool compute,
                 cudaStream_t s) {
  CeTransport& ce = *cm->ce;
  const int P = p.P, me = cm->rank, n = p.n, d = p.d;
  const auto& peer_ws = ce.peers(ws, s, p.peer_key);
  if (cm->sched) sched_a2a_begin(cm, s);
  for (int src = 0; src < P; ++src) {
    cudaStream_t st = ce.disp_stream(src);
    LINA_CUDA_CHECK(cudaStreamWaitEvent(st, e_cb, 0));
    if (src != me) ce.wait_flag(st, CeTransport::kReadyBwdD, src, 0, seq);
    for (int c = 0; c < n; ++c) {
      LINA_CUDA_CHECK(cudaMemcpyAsync(q.dO + recv_block(p, c, src, d), peer_ws[src] + p.w_dS + send_block(p, c, me, d),
                                      block_bytes(p, d), cudaMemcpyDeviceToDevice, st));
      LINA_CUDA_CHECK(cudaEventRecord(ce.ev(0, src, c), st));
    }
    if (src != me) ce.post_flag(st, src, CeTransport::kPulledBwdD, me, 0, seq);
  }
  for (int r = 0; r < P; ++r)  // every peer has pulled my previous dXe
    if (r != me) ce.wait_flag(s, CeTransport::kPulledBwdC, r, 0, ce.prev_ce_bwd);
  for (int c = 0; c < n; ++c) {
    for (int src = 0; src < P; ++src) LINA_CUDA_CHECK(cudaStreamWaitEvent(s, ce.ev(0, src, c), 0));
    if (compute) {
      prof_begin(cm, s);
      row_gemm(p, q.dO, w2, q.dH, q.H, q.vcount, q.mtp, c, p.f, p.d, false, kEpiMask, s, nullptr, q.mask);
      row_gemm(p, q.dH, w1, q.dXe, nullptr, q.vcount, q.mtp, c, p.d, p.f, false, kEpiNone, s);
      prof_end(cm, s, 2);
    }
    for (int r = 0; r < P; ++r)
      if (r != me) ce.post_flag(s, r, CeTransport::kReadyBwdC, me, c, seq);
    LINA_CUDA_CHECK(cudaEventRecord(ce.ev(1, me, c), s));
  }
  for (int src = 0; src < P; ++src) {
    cudaStream_t st = ce.comb_stream(src);
    LINA_CUDA_CHECK(cudaStreamWaitEvent(st, e_cb, 0));
    for (int c = 0; c < n; ++c) {
      if (src == me) LINA_CUDA_CHECK(cudaStreamWaitEvent(st, ce.ev(1, me, c), 0));
      else ce.wait_flag(st, CeTransport::kReadyBwdC, src, c, seq);
      LINA_CUDA_CHECK(cudaMemcpyAsync(q.dXs + send_block(p, c, src, d), peer_ws[src] + p.w_dXe + recv_block(p, c, me, d),
                                      block_bytes(p, d), cudaMemcpyDeviceToDevice, st));
    }
    if (src != me) ce.post_flag(st, src, CeTransport::kPulledBwdC, me, 0, seq);
    LINA_CUDA_CHECK(cudaEventRecord(ce.ev(2, src, CeTransport::kMaxChunks), st));
    if (cm->sched) sched_a2a_end(cm, st);
  }
  // weight gradients overlap the last combine pulls
  WGrad wg2{q.dO, q.H, dw2, q.vcount, n, P, p.El, p.Cm, p.d, p.f};
  WGrad wg1{q.dH, q.R, dw1, q.vcount, n, P, p.El, p.Cm, p.f, p.d};
  if (compute) {
    prof_begin(cm, s);
    launch_expert_wgrad(dtype, wg2, s);
    launch_expert_wgrad(dtype, wg1, s);
    prof_end(cm, s, 2);
  }
  for (int src = 0; src < P; ++src)
    LINA_CUDA_CHECK(cudaStreamWaitEvent(s, ce.ev(2, src, CeTransport::kMaxChunks), 0));
}

// ------------------------------------------------------------------ fused transport
// The all-to-alls disappear into the kernels that produce their data (NVLink 5 peer
// stores through IPC-mapped buffers): permute / combine-backward store each row into
// its owner's receive buffer; the GEMM2 / dgrad2 epilogues TMA-store each output tile
// into the owner's send-layout buffer while the tensor cores work on the next tile.
// Cross-rank ordering (signal.h): FREE (this rank's receive buffers of the round may be
// written) and READY (a rank's stores of the round are complete) are release stores of
// the round number into the peers' flag slots, made by the kernels themselves — FREE
// by the first kernel after the buffers' last reader, READY by the last CTA of the
// producing kernel — and acquired by the first consuming kernel (one spinning thread
// per CTA).  No stream memory operation and no extra launch on the critical path.
// Signal of one kernel: wait for `wait_kind` at *wait_round + wait_add, publish `post_kind`
// at *post_round + post_add, optionally close the pass's round (bump) in its last CTA.
PeerSignal make_sig(lina_comm* cm, int wait_kind, const uint32_t* wait_round, uint32_t wait_add, int post_kind,
                    const uint32_t* post_round, uint32_t post_add, int done_site = -1, uint32_t* bump = nullptr) {
  CeTransport& ce = *cm->ce;
  PeerSignal g;
  g.P = cm->world;
  g.me = cm->rank;
  g.stride = CeTransport::kMaxChunks;
  if (wait_kind >= 0) {
    g.wait = ce.slots(wait_kind);
    g.wait_round = wait_round;
    g.wait_add = wait_add;
  }
  if (post_kind >= 0) {
    g.post = ce.peer_slots(post_kind);
    g.post_round = post_round;
    g.post_add = post_add;
  }
  g.done = done_site >= 0 ? ce.done_counter(done_site) : nullptr;
  g.bump = bump;
  return g;
}
// The wait part of a signal runs as its own 1-CTA kernel (launch_sig_wait); the consumer
// gets the rest.
PeerSignal wait_only(PeerSignal g) {
  g.post = nullptr;
  g.bump = nullptr;
  g.done = nullptr;
  return g;
}
PeerSignal no_wait(PeerSignal g) {
  g.wait = nullptr;
  g.wait_round = nullptr;
  return g;
}
enum { kSiteDispFwd = 0, kSiteCombFwd = 1, kSiteDispBwd = 2, kSiteCombBwd = 3, kSiteFwdEnd = 4, kSiteBwdEnd = 5 };

bool fused_ok(const lina_comm* cm, const Plan& p) {
  return cm->transport == 2 && cm->ce && p.P > 1 && p.bf16 && p.d % 256 == 0 && p.f % 256 == 0 &&
         p.d % 64 == 0 && p.f % 64 == 0 && p.d % 32 == 0;
}

// Split dispatch (n = 1; permute.cu split_rows_kernel, gemm_tc.cu src_wait): the counts go
// first (one 1-CTA kernel), this rank's own rows move on the compute stream, the peers' rows
// on the high-priority stream by a persistent grid of LINA_DISPATCH_CTAS CTAs (default: one
// per SM) that shares the SMs with the expert GEMM, posting READY per owner; the owner's
// GEMM1 / dgrad1 start on its own source's rows and take a peer's rows once that peer has
// posted them ("the expert can start computing with a subset of the tokens").
// LINA_SPLIT_DISPATCH=0: the whole dispatch before the GEMMs (round-1 order).
bool split_dispatch(const Plan& p) {
  static const bool on = [] {
    const char* e = getenv("LINA_SPLIT_DISPATCH");
    return !(e && e[0] == '0');
  }();
  return on && p.n == 1 && p.P <= 8;
}
int split_ctas() {
  static const int n = [] {
    const char* e = getenv("LINA_DISPATCH_CTAS");
    if (e && atoi(e) > 0) return atoi(e);
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
  }();
  return n;
}
enum { kSiteSplitFwd = 16, kSiteSplitBwd = 24 };
// LINA_SCHED_WINDOW=dispatch (split dispatch only): the all-to-all phase the allreduce
// scheduler defers to is the peer-row dispatch kernel alone, not the expert GEMMs whose
// epilogues return the rows (a B200 reading of "no all-to-all in flight": there the
// link traffic is the dispatch; the return is spread over dgrad2's tiles).  Default: the
// whole window from combine-backward to the last returned tile.
bool sched_window_dispatch() {
  static const bool on = [] {
    const char* e = getenv("LINA_SCHED_WINDOW");
    return e && std::string(e) == "dispatch";
  }();
  return on;
}

// Micro-op c of a signal: slot c of the kind (wait: chunks [c, c + wait_chunks)).
PeerSignal chunk_sig(PeerSignal g, int c, int wait_chunks = 1) {
  if (g.wait) g.wait += c;
  g.wait_chunks = wait_chunks;
  g.post_chunk = c;
  return g;
}

// Host-side cached per-rank tensor maps of a peer-stored GEMM output.
PeerStore peer_store(CeTransport& ce, const char* tag, void* buf, size_t off, const Plan& p, int me,
                     std::vector<char*>& bases, cudaStream_t s) {
  const auto& ps = ce.peers(buf, s, p.peer_key);
  bases.resize(p.P);
  for (int r = 0; r < p.P; ++r) bases[r] = ps[r] + off;
  PeerStore st;
  const std::string key = std::string(tag) + std::to_string((uintptr_t)buf) + "@" +
                          std::to_string(ce.generation(buf)) + ":" + std::to_string(off) + ":" +
                          std::to_string(p.Cm) + ":" + std::to_string(p.n * p.E);
  auto it = ce.host_blobs.find(key);
  if (it == ce.host_blobs.end()) it = ce.host_blobs.emplace(key, tc_peer_dmaps(bases, p.d, p.Cm, p.n * p.E)).first;
  st.host_maps = it->second.data();
  st.bases = bases.data();
  st.P = p.P;
  st.me = me;
  st.E = p.E;
  return st;
}

RowGemm peer_gemm(const Plan& p, const void* A, const void* B, void* D, const int* vcount, const int* mtp, int c,
                  int N, int K) {
  RowGemm g{};
  g.tile_rows = p.tile_rows;
  g.half_tails = p.half_tails;
  g.mtp = mtp + (size_t)c * (p.P * p.El + 1);
  g.A = A;
  g.B = B;
  g.D = D;
  g.vcount = vcount;
  g.seg0 = c * p.P * p.El;
  g.nseg = p.P * p.El;
  g.El = p.El;
  g.Cm = p.Cm;
  g.N = N;
  g.K = K;
  set_tail(p, g, mtp, c);
  return g;
}

// n = 1: everything on the caller's stream.  n > 1 (the paper's micro-op pipeline,
// P:354-376): the data-movement kernels of micro-op c + 1 run on the high-priority
// stream while the expert GEMMs of micro-op c run on the caller's stream (they share
// the SMs: the movers need no shared memory), each micro-op with its own flag slot.
void forward_fused(lina_comm* cm, const Plan& p, const Ptrs& q, const void* tokens, const float* gate_w,
                   const void* w1, const void* w2, void* out, void* saved, void* ws, lina_route* route,
                   cudaStream_t s) {
  using CT = CeTransport;
  CeTransport& ce = *cm->ce;
  const int dtype = 1, P = p.P, me = cm->rank, n = p.n;
  const bool override_r = route && route->override_routing;
  uint32_t* rf = ce.round_fwd();  // this forward's round is *rf + 1 (closed by the combine kernel)
  trace_mark(cm, s, "fwd:start");
  if (override_r) {
    LINA_CUDA_CHECK(cudaMemcpyAsync(q.idx, route->idx, 4 * (size_t)p.T * p.k, cudaMemcpyDeviceToDevice, s));
    LINA_CUDA_CHECK(cudaMemcpyAsync(q.gate, route->gate, 4 * (size_t)p.T * p.k, cudaMemcpyDeviceToDevice, s));
  }
  // gate: block 0 posts FREE (my R, recv counts and Cb were last read by the previous backward)
  const PeerSignal s_free = make_sig(cm, -1, nullptr, 0, CT::kFreeFwd, rf, 1);
  launch_gate_topk(dtype, tokens, gate_w, p.T, p.d, p.E, p.k, override_r ? 0 : 1, q.probs, q.idx, q.gate, s,
                   &s_free);
  launch_route(q.idx, p.T, p.k, p.E, p.C, q.route, q.slot, route ? route->counts : nullptr, q.kept,
               q.tok_of, s, cm->route_sync);
  trace_mark(cm, s, "gate+route");
  void* const* peer_R = ce.dev_ptrs(saved, p.s_R, s, p.peer_key);
  void* const* peer_cnt = ce.dev_ptrs(saved, p.s_recvkept, s, p.peer_key);
  std::vector<char*> cb;
  const PeerStore st = peer_store(ce, "fwdC:", saved, p.s_C, p, me, cb, s);
  // dispatch = permute into the owners' R (after their FREE; READY per micro-op)
  const PeerSignal s_disp = make_sig(cm, CT::kFreeFwd, rf, 1, CT::kFReadyFwdD, rf, 1, kSiteDispFwd);
  const bool split = split_dispatch(p);
  cudaStream_t sm = (n > 1 || split) ? cm->hi : s;  // the mover stream
  if (split) {
    // counts first (after the owners' FREE), then the peers' rows on `hi` beside GEMM1
    launch_dispatch_counts(q.kept, P, p.El, me, peer_cnt, wait_only(s_disp),
                           make_sig(cm, -1, nullptr, 0, CT::kFCountFwdS, rf, 1), s);
    LINA_CUDA_CHECK(cudaEventRecord(cm->ev[0], s));
    LINA_CUDA_CHECK(cudaStreamWaitEvent(sm, cm->ev[0], 0));
    prof_a2a_begin(cm, sm);
    launch_permute_split(dtype, tokens, q.tok_of, q.kept, p.k, p.d, p.E, p.C, p.Cm, p.El, P, me, peer_R, 1, P - 1,
                         split_ctas(), make_sig(cm, -1, nullptr, 0, CT::kFReadyFwdD, rf, 1),
                         ce.done_counter(kSiteSplitFwd), sm);
    LINA_CUDA_CHECK(cudaEventRecord(cm->ev[1], sm));
    launch_permute_split(dtype, tokens, q.tok_of, q.kept, p.k, p.d, p.E, p.C, p.Cm, p.El, P, me, peer_R, 0, 1, 0,
                         PeerSignal{}, nullptr, s);  // this rank's own rows
  } else {
    if (n > 1) {
      LINA_CUDA_CHECK(cudaEventRecord(cm->ev[0], s));
      LINA_CUDA_CHECK(cudaStreamWaitEvent(sm, cm->ev[0], 0));
    }
    prof_a2a_begin(cm, sm);
    launch_sig_wait(wait_only(s_disp), sm);
    for (int c = 0; c < n; ++c)
      launch_permute_peer(dtype, tokens, q.tok_of, q.kept, p.k, p.d, p.E, p.C, c, 1, p.Cm, p.El, P, me, peer_R,
                          peer_cnt, chunk_sig(no_wait(s_disp), c), sm);
    if (n > 1) LINA_CUDA_CHECK(cudaEventRecord(cm->ev[1], sm));
  }
  trace_mark(cm, s, "permute(peer)");
  if (route) {
    if (route->idx && !override_r)
      LINA_CUDA_CHECK(cudaMemcpyAsync(route->idx, q.idx, 4 * (size_t)p.T * p.k, cudaMemcpyDeviceToDevice, s));
    if (route->gate && !override_r)
      LINA_CUDA_CHECK(cudaMemcpyAsync(route->gate, q.gate, 4 * (size_t)p.T * p.k, cudaMemcpyDeviceToDevice, s));
    if (route->slot)
      LINA_CUDA_CHECK(cudaMemcpyAsync(route->slot, q.slot, 4 * (size_t)p.T * p.k, cudaMemcpyDeviceToDevice, s));
    if (route->probs)
      LINA_CUDA_CHECK(cudaMemcpyAsync(route->probs, q.probs, 4 * (size_t)p.T * p.E, cudaMemcpyDeviceToDevice, s));
  }
  const PeerSignal s_recv = make_sig(cm, CT::kFReadyFwdD, rf, 1, -1, nullptr, 0);
  const PeerSignal s_comb = make_sig(cm, -1, nullptr, 0, CT::kFReadyFwdC, rf, 1, kSiteCombFwd);
  for (int c = 0; c < n; ++c) {
    if (split)  // every source's counts have landed (its rows follow: GEMM1 waits per source)
      launch_sig_wait(wait_only(make_sig(cm, CT::kFCountFwdS, rf, 1, -1, nullptr, 0)), s);
    else
      launch_sig_wait(wait_only(chunk_sig(s_recv, c)), s);  // micro-op c (and with c = 0 the counts) has landed
    if (c == 0) {
      launch_vcount(q.recv_kept, P, p.El, p.C, n, q.vcount, s);
      launch_mtile_prefix(q.vcount, n, P * p.El, p.tile_rows, q.mtp, s);
      tile_lists(p, q, s);
      trace_mark(cm, s, "vcount");
      prof_begin(cm, s);
    }
    if (split)
      row_gemm(p, q.R, w1, q.H, nullptr, q.vcount, q.mtp, c, p.f, p.d, true, kEpiRelu, s, q.mask, nullptr, &s_recv,
               me);
    else
      row_gemm(p, q.R, w1, q.H, nullptr, q.vcount, q.mtp, c, p.f, p.d, true, kEpiRelu, s, q.mask);
    trace_mark(cm, s, "gemm1");
    RowGemm g = peer_gemm(p, q.H, w2, q.O, q.vcount, q.mtp, c, p.d, p.f);
    const PeerSignal s_c = chunk_sig(s_comb, c);
    g.sig = &s_c;  // the last CTA posts READY of micro-op c
    launch_row_gemm_tc_peer(g, true, kEpiNone, st, s);  // combine all-to-all in the epilogue
    trace_mark(cm, s, "gemm2(peer)");
  }
  prof_end(cm, s, 2 * n);
  if (n > 1 || split) LINA_CUDA_CHECK(cudaStreamWaitEvent(s, cm->ev[1], 0));  // join the mover stream
  // combine: the returned expert outputs of every micro-op have landed (1-CTA wait); its
  // last CTA closes the forward's round
  const PeerSignal s_out = make_sig(cm, CT::kFReadyFwdC, rf, 1, -1, nullptr, 0, kSiteFwdEnd, rf);
  launch_sig_wait(wait_only(chunk_sig(s_out, 0, n)), s);
  prof_a2a_end(cm, s);
  const PeerSignal s_out2 = no_wait(s_out);
  launch_combine(dtype, q.Cb, q.idx, q.slot, q.gate, p.T, p.k, p.d, p.E, p.C, n, p.Cm, out, s, &s_out2);
  trace_mark(cm, s, "combine");
}

void backward_fused(lina_comm* cm, const Plan& p, const Ptrs& q, const void* dout, const void* tokens,
                    const float* gate_w, const void* w1, const void* w2, void* dtokens, float* dgate_w,
                    void* dw1, void* dw2, void* ws, cudaStream_t s) {
  using CT = CeTransport;
  CeTransport& ce = *cm->ce;
  const int dtype = 1, P = p.P, me = cm->rank, n = p.n;
  uint32_t* rf = ce.round_fwd();  // the last forward's round (closed)
  uint32_t* rb = ce.round_bwd();  // this backward's round is *rb + 1 (closed by the dX kernel)
  trace_mark(cm, s, "bwd:start");
  void* const* peer_dO = ce.dev_ptrs(ws, p.w_dO, s, p.peer_key);
  std::vector<char*> dxs;
  const PeerStore st = peer_store(ce, "bwdC:", ws, p.w_dXs, p, me, dxs, s);
  if (cm->sched) sched_a2a_imminent(cm, s);
  // backward dispatch = combine-backward into the owners' dO (after the backward FREE they
  // posted at the end of their previous backward, once its wgrad and dX had read dO and
  // dXs — so layers sharing one workspace on a comm stay ordered; READY per micro-op)
  const PeerSignal s_disp = make_sig(cm, CT::kFreeBwd, rb, 0, CT::kFReadyBwdD, rb, 1, kSiteDispBwd);
  const bool split = split_dispatch(p);
  cudaStream_t sm = (n > 1 || split) ? cm->hi : s;
  if (split) {
    // the peers' rows on `hi` (every CTA first waits for the owners' backward FREE), this
    // rank's own rows on `s`; dg of dropped assignments stays 0
    if (p.T > 0) LINA_CUDA_CHECK(cudaMemsetAsync(q.dg, 0, sizeof(float) * (size_t)p.T * p.k, s));
    LINA_CUDA_CHECK(cudaEventRecord(cm->ev[2], s));
    LINA_CUDA_CHECK(cudaStreamWaitEvent(sm, cm->ev[2], 0));
    prof_a2a_begin(cm, sm);
    PeerSignal s_rows = make_sig(cm, CT::kFreeBwd, rb, 0, CT::kFReadyBwdD, rb, 1);
    launch_combine_bwd_split(dtype, dout, q.Cb, q.tok_of, q.kept, q.gate, p.k, p.d, p.E, p.C, p.Cm, p.El, P, me,
                             peer_dO, q.dg, 1, P - 1, split_ctas(), s_rows, ce.done_counter(kSiteSplitBwd), sm);
    if (cm->sched && sched_window_dispatch()) sched_a2a_end(cm, sm);
    LINA_CUDA_CHECK(cudaEventRecord(cm->ev[3], sm));
    launch_combine_bwd_split(dtype, dout, q.Cb, q.tok_of, q.kept, q.gate, p.k, p.d, p.E, p.C, p.Cm, p.El, P, me,
                             peer_dO, q.dg, 0, 1, 0, PeerSignal{}, nullptr, s);  // this rank's own rows
  } else {
    if (n > 1) {
      LINA_CUDA_CHECK(cudaEventRecord(cm->ev[2], s));
      LINA_CUDA_CHECK(cudaStreamWaitEvent(sm, cm->ev[2], 0));
    }
    prof_a2a_begin(cm, sm);
    launch_sig_wait(wait_only(s_disp), sm);
    for (int c = 0; c < n; ++c)
      launch_combine_bwd_peer(dtype, dout, q.Cb, q.tok_of, q.kept, q.gate, p.T, p.k, p.d, p.E, p.C, c, 1, p.Cm,
                              p.El, P, me, peer_dO, q.dg, chunk_sig(no_wait(s_disp), c), sm);
    if (n > 1) LINA_CUDA_CHECK(cudaEventRecord(cm->ev[3], sm));
  }
  trace_mark(cm, s, "combine_bwd(peer)");
  const PeerSignal s_recv = make_sig(cm, CT::kFReadyBwdD, rb, 1, -1, nullptr, 0);
  const PeerSignal s_comb = make_sig(cm, -1, nullptr, 0, CT::kFReadyBwdC, rb, 1, kSiteCombBwd);
  prof_begin(cm, s);
  for (int c = 0; c < n; ++c) {
    if (split) {  // dgrad1 takes each source's dO rows as soon as that source has posted them
      row_gemm(p, q.dO, w2, q.dH, q.H, q.vcount, q.mtp, c, p.f, p.d, false, kEpiMask, s, nullptr, q.mask, &s_recv,
               me);
    } else {
      launch_sig_wait(wait_only(chunk_sig(s_recv, c)), s);  // micro-op c of the peers' dO rows has landed
      row_gemm(p, q.dO, w2, q.dH, q.H, q.vcount, q.mtp, c, p.f, p.d, false, kEpiMask, s, nullptr, q.mask);
    }
    trace_mark(cm, s, "dgrad1");
    RowGemm g = peer_gemm(p, q.dH, w1, q.dXe, q.vcount, q.mtp, c, p.d, p.f);
    const PeerSignal s_c = chunk_sig(s_comb, c);
    g.sig = &s_c;
    launch_row_gemm_tc_peer(g, false, kEpiNone, st, s);  // combine all-to-all in the epilogue
    trace_mark(cm, s, "dgrad2(peer)");
  }
  // the last kernel that moves all-to-all bytes is done: allreduce micro-ops may run
  // beside the weight gradients, dWg and dX (compute only)
  if (cm->sched && !(split && sched_window_dispatch())) sched_a2a_end(cm, s);
  WGrad wg2{q.dO, q.H, dw2, q.vcount, n, P, p.El, p.Cm, p.d, p.f};
  WGrad wg1{q.dH, q.R, dw1, q.vcount, n, P, p.El, p.Cm, p.f, p.d};
  launch_expert_wgrad(dtype, wg2, s);
  launch_expert_wgrad(dtype, wg1, s);
  prof_end(cm, s, 2 * n + 2);
  trace_mark(cm, s, "wgrad x2");
  if (n > 1 || split) LINA_CUDA_CHECK(cudaStreamWaitEvent(s, cm->ev[3], 0));  // dg of every micro-op
  // dWg needs only this rank's dg: it overlaps the last returning expert gradients
  launch_dwg(dtype, tokens, q.probs, q.idx, q.gate, q.dg, p.T, p.d, p.E, p.k, q.dwg, dgate_w, s);
  trace_mark(cm, s, "dwg");
  const PeerSignal s_back = make_sig(cm, CT::kFReadyBwdC, rb, 1, -1, nullptr, 0, kSiteBwdEnd, rb);
  launch_sig_wait(wait_only(chunk_sig(s_back, 0, n)), s);
  prof_a2a_end(cm, s);
  const PeerSignal s_back2 = no_wait(s_back);
  launch_dx(dtype, q.dXs, q.idx, q.slot, q.probs, q.gate, q.dg, gate_w, p.T, p.k, p.d, p.E, p.C, n, p.Cm,
            dtokens, s, &s_back2, nullptr, q.dwg);
  // backward FREE: my dO and dXs have been read (wgrad, dX) — publish the round just closed
  launch_sig_wait(make_sig(cm, -1, nullptr, 0, CT::kFreeBwd, rb, 0), s);
  trace_mark(cm, s, "dx");
}

// Collectives-only passes of the fused transport (lina_profile_enable flag 4; SURVEY.md
// §8(d) T_a2a(n)): the 2n all-to-all micro-ops of a pass with their in-kernel signals and
// nothing else — the dispatch kernel (permute / combine-backward peer stores, as in the
// real pass) and, for the return all-to-all that the real pass folds into the GEMM2 /
// dgrad2 epilogues, a stand-alone mover of the same rows.  Routing (tok_of, kept, gate)
// is the last real forward's, from `saved`.  All on the caller's stream, in order.
void forward_fused_movers(lina_comm* cm, const Plan& p, const Ptrs& q, const void* tokens, void* saved,
                          cudaStream_t s) {
  using CT = CeTransport;
  CeTransport& ce = *cm->ce;
  const int dtype = 1, P = p.P, me = cm->rank, n = p.n;
  uint32_t* rf = ce.round_fwd();
  launch_sig_wait(make_sig(cm, -1, nullptr, 0, CT::kFreeFwd, rf, 1), s);  // (the gate kernel posts it normally)
  void* const* peer_R = ce.dev_ptrs(saved, p.s_R, s, p.peer_key);
  void* const* peer_cnt = ce.dev_ptrs(saved, p.s_recvkept, s, p.peer_key);
  void* const* peer_C = ce.dev_ptrs(saved, p.s_C, s, p.peer_key);
  const PeerSignal s_disp = make_sig(cm, CT::kFreeFwd, rf, 1, CT::kFReadyFwdD, rf, 1, kSiteDispFwd);
  launch_sig_wait(wait_only(s_disp), s);
  for (int c = 0; c < n; ++c)
    launch_permute_peer(dtype, tokens, q.tok_of, q.kept, p.k, p.d, p.E, p.C, c, 1, p.Cm, p.El, P, me, peer_R,
                        peer_cnt, chunk_sig(no_wait(s_disp), c), s);
  const PeerSignal s_recv = make_sig(cm, CT::kFReadyFwdD, rf, 1, -1, nullptr, 0);
  const PeerSignal s_comb = make_sig(cm, -1, nullptr, 0, CT::kFReadyFwdC, rf, 1, kSiteCombFwd);
  for (int c = 0; c < n; ++c) {
    launch_sig_wait(wait_only(chunk_sig(s_recv, c)), s);
    if (c == 0) launch_vcount(q.recv_kept, P, p.El, p.C, n, q.vcount, s);
    launch_push_segments(dtype, q.O, peer_C, q.vcount, c, P, p.El, p.E, p.Cm, me, p.d, chunk_sig(s_comb, c), s);
  }
  // every returned micro-op has landed; close the forward's round
  launch_sig_wait(chunk_sig(make_sig(cm, CT::kFReadyFwdC, rf, 1, -1, nullptr, 0, -1, rf), 0, n), s);
}

void backward_fused_movers(lina_comm* cm, const Plan& p, const Ptrs& q, const void* dout, void* ws,
                           cudaStream_t s) {
  using CT = CeTransport;
  CeTransport& ce = *cm->ce;
  const int dtype = 1, P = p.P, me = cm->rank, n = p.n;
  uint32_t* rb = ce.round_bwd();
  void* const* peer_dO = ce.dev_ptrs(ws, p.w_dO, s, p.peer_key);
  void* const* peer_dXs = ce.dev_ptrs(ws, p.w_dXs, s, p.peer_key);
  const PeerSignal s_disp = make_sig(cm, CT::kFreeBwd, rb, 0, CT::kFReadyBwdD, rb, 1, kSiteDispBwd);
  launch_sig_wait(wait_only(s_disp), s);
  for (int c = 0; c < n; ++c)
    launch_combine_bwd_peer(dtype, dout, q.Cb, q.tok_of, q.kept, q.gate, p.T, p.k, p.d, p.E, p.C, c, 1, p.Cm, p.El,
                            P, me, peer_dO, q.dg, chunk_sig(no_wait(s_disp), c), s);
  const PeerSignal s_recv = make_sig(cm, CT::kFReadyBwdD, rb, 1, -1, nullptr, 0);
  const PeerSignal s_comb = make_sig(cm, -1, nullptr, 0, CT::kFReadyBwdC, rb, 1, kSiteCombBwd);
  for (int c = 0; c < n; ++c) {
    launch_sig_wait(wait_only(chunk_sig(s_recv, c)), s);
    launch_push_segments(dtype, q.dXe, peer_dXs, q.vcount, c, P, p.El, p.E, p.Cm, me, p.d, chunk_sig(s_comb, c), s);
  }
  launch_sig_wait(chunk_sig(make_sig(cm, CT::kFReadyBwdC, rb, 1, -1, nullptr, 0, -1, rb), 0, n), s);
  launch_sig_wait(make_sig(cm, -1, nullptr, 0, CT::kFreeBwd, rb, 0), s);  // backward FREE
}

// ------------------------------------------------------------------ dropless layout
// (§8(f) row 4; kernels/dropless.cu): no capacity bound, a count exchange, unequal-split
// dispatch / return by peer stores, the expert GEMMs over virtual segments.  n_chunks = 1.
// Communicator of this rank's packing group (ranks [G·m, (G+1)·m)), split off the dispatch
// communicator on first use (collective: every rank reaches it in the same call).
ncclComm_t group_comm(lina_comm* cm, int m) {
  auto it = cm->group_comms.find(m);
  if (it != cm->group_comms.end()) return it->second;
  if (!cm->ep_disp)
    throw StatusError{LINA_ERR_UNSUPPORTED, "expert packing needs an NCCL communicator (lina_comm_init)"};
  ncclComm_t g = nullptr;
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  LINA_NCCL_CHECK(ncclCommSplit(cm->ep_disp, cm->rank / m, cm->rank, &g, &cfg));
  cm->group_comms[m] = g;
  return g;
}

RowGemm dl_gemm(const Plan& p, const Ptrs& q, const void* A, const void* B, void* D, int N, int K) {
  RowGemm g{};
  g.tile_rows = p.tile_rows;
  g.half_tails = p.half_tails;
  g.A = A;
  g.B = B;
  g.D = D;
  g.vcount = q.dl.vcount;
  g.mtp = q.dl.mtp;
  g.seg0 = 0;
  g.nseg = p.V;
  g.El = p.V;               // segment v's weight index = seg_expert[v % V] = vexp[v]
  g.seg_expert = q.dl.vexp;
  g.B_experts = p.El;
  g.Cm = p.tile_rows;
  g.N = N;
  g.K = K;
  if (p.tail_split) g.mtp_tail = q.dl.mtpt;  // segments of <= 128 rows as single-CTA tiles (row base 0)
  return g;
}

void forward_dropless(lina_comm* cm, const Plan& p, const Ptrs& q, const void* tokens, const float* gate_w,
                      const void* w1, const void* w2, void* out, void* saved, lina_route* route, cudaStream_t s) {
  using CT = CeTransport;
  const int dtype = p.bf16 ? 1 : 0, P = p.P, me = cm->rank, E = p.E, El = p.El, R = p.tile_rows;
  const bool peer = P > 1;
  CeTransport* ce = peer ? cm->ce : nullptr;
  uint32_t* rf = peer ? ce->round_fwd() : nullptr;
  const bool override_r = route && route->override_routing;
  trace_mark(cm, s, "dl fwd:start");
  if (override_r) {
    LINA_CUDA_CHECK(cudaMemcpyAsync(q.idx, route->idx, 4 * (size_t)p.T * p.k, cudaMemcpyDeviceToDevice, s));
    LINA_CUDA_CHECK(cudaMemcpyAsync(q.gate, route->gate, 4 * (size_t)p.T * p.k, cudaMemcpyDeviceToDevice, s));
  }
  // gate (block 0 posts FREE: my R, counts and returned rows were last read by the previous backward)
  const PeerSignal s_free = peer ? make_sig(cm, -1, nullptr, 0, CT::kFreeFwd, rf, 1) : PeerSignal{};
  launch_gate_topk(dtype, tokens, gate_w, p.T, p.d, E, p.k, override_r ? 0 : 1, q.probs, q.idx, q.gate, s,
                   peer ? &s_free : nullptr);
  launch_route(q.idx, p.T, p.k, E, p.C, q.route, q.slot, route ? route->counts : nullptr, q.kept, q.tok_of, s,
               cm->route_sync);
  if (p.pack > 1) group_comm(cm, p.pack);  // (created by the first, eager call)
  const int* allc = q.kept;
  if (peer) {  // the count exchange, then every rank derives the same layout
    prof_a2a_begin(cm, s);
    prof_comm_begin(cm, s);
    int* const* peer_allc = (int* const*)ce->dev_ptrs(saved, p.s_allc, s, p.peer_key);
    launch_dl_counts(q.kept, peer_allc, P, me, E, make_sig(cm, CT::kFreeFwd, rf, 1, CT::kFCountFwd, rf, 1), s);
    launch_sig_wait(make_sig(cm, CT::kFCountFwd, rf, 1, -1, nullptr, 0), s);
    allc = q.allc;
  }
  launch_dl_layout(allc, P, E, El, p.pack, me, R, p.V, p.tail_split ? 1 : 0, q.dl, s);
  trace_mark(cm, s, "dl gate+route+layout");
  if (peer) {
    void* const* peer_R = ce->dev_ptrs(saved, p.s_R, s, p.peer_key);
    launch_dl_permute(dtype, tokens, q.tok_of, q.kept, q.dl, me, p.T, p.C, p.k, E, El, p.pack, p.d, peer_R, nullptr,
                      make_sig(cm, -1, nullptr, 0, CT::kFReadyFwdD, rf, 1, kSiteDispFwd), s);
    launch_sig_wait(make_sig(cm, CT::kFReadyFwdD, rf, 1, -1, nullptr, 0), s);  // every source's rows landed
    prof_comm_end(cm, s);
  } else {
    launch_dl_permute(dtype, tokens, q.tok_of, q.kept, q.dl, me, p.T, p.C, p.k, E, El, 1, p.d, nullptr, q.R, PeerSignal{},
                      s);
  }
  if (route) {
    if (route->idx && !override_r)
      LINA_CUDA_CHECK(cudaMemcpyAsync(route->idx, q.idx, 4 * (size_t)p.T * p.k, cudaMemcpyDeviceToDevice, s));
    if (route->gate && !override_r)
      LINA_CUDA_CHECK(cudaMemcpyAsync(route->gate, q.gate, 4 * (size_t)p.T * p.k, cudaMemcpyDeviceToDevice, s));
    if (route->slot)
      LINA_CUDA_CHECK(cudaMemcpyAsync(route->slot, q.slot, 4 * (size_t)p.T * p.k, cudaMemcpyDeviceToDevice, s));
    if (route->probs)
      LINA_CUDA_CHECK(cudaMemcpyAsync(route->probs, q.probs, 4 * (size_t)p.T * E, cudaMemcpyDeviceToDevice, s));
  }
  trace_mark(cm, s, "dl dispatch");
  prof_begin(cm, s);
  RowGemm g1 = dl_gemm(p, q, q.R, w1, q.H, p.f, p.d);
  g1.mask_out = q.mask;
  launch_expert_row_gemm(dtype, g1, true, kEpiRelu, s);
  launch_expert_row_gemm(dtype, dl_gemm(p, q, q.H, w2, q.O, p.d, p.f), true, kEpiNone, s);
  prof_end(cm, s, 2);
  trace_mark(cm, s, "dl gemm1+gemm2");
  if (peer) {  // return all-to-all: each segment's rows to its source's compact buffer
    void* const* peer_C = ce->dev_ptrs(saved, p.s_C, s, p.peer_key);
    prof_comm_begin(cm, s);
    launch_dl_push_vsegs(dtype, q.O, peer_C, q.dl, p.V, R, E, El, p.pack, me, p.d,
                         make_sig(cm, -1, nullptr, 0, CT::kFReadyFwdC, rf, 1, kSiteCombFwd), s);
    const PeerSignal s_out = make_sig(cm, CT::kFReadyFwdC, rf, 1, -1, nullptr, 0, kSiteFwdEnd, rf);
    launch_sig_wait(wait_only(s_out), s);
    prof_comm_end(cm, s);
    prof_a2a_end(cm, s);
    const PeerSignal s_out2 = no_wait(s_out);
    launch_combine(dtype, q.Cb, q.idx, q.slot, q.gate, p.T, p.k, p.d, E, p.C, 1, p.C, out, s, &s_out2, q.dl.ebase);
  } else {
    launch_combine(dtype, q.O, q.idx, q.slot, q.gate, p.T, p.k, p.d, E, p.C, 1, p.C, out, s, nullptr, q.dl.ebase);
  }
  trace_mark(cm, s, "dl combine");
}

void backward_dropless(lina_comm* cm, const Plan& p, const Ptrs& q, const void* dout, const void* tokens,
                       const float* gate_w, const void* w1, const void* w2, void* dtokens, float* dgate_w, void* dw1,
                       void* dw2, void* ws, cudaStream_t s) {
  using CT = CeTransport;
  const int dtype = p.bf16 ? 1 : 0, P = p.P, me = cm->rank, E = p.E, El = p.El, R = p.tile_rows;
  const bool peer = P > 1;
  CeTransport* ce = peer ? cm->ce : nullptr;
  uint32_t* rb = peer ? ce->round_bwd() : nullptr;
  trace_mark(cm, s, "dl bwd:start");
  if (cm->sched) sched_a2a_imminent(cm, s);
  const void* O = peer ? (const void*)q.Cb : (const void*)q.O;  // the returned expert outputs
  // dg = 0 for assignments a capacity bound dropped (the row kernel writes the kept ones)
  if (p.C < p.T && p.T > 0) LINA_CUDA_CHECK(cudaMemsetAsync(q.dg, 0, sizeof(float) * (size_t)p.T * p.k, s));
  if (peer) {
    prof_a2a_begin(cm, s);
    const PeerSignal s_disp = make_sig(cm, CT::kFreeBwd, rb, 0, CT::kFReadyBwdD, rb, 1, kSiteDispBwd);
    launch_sig_wait(wait_only(s_disp), s);
    prof_comm_begin(cm, s);
    void* const* peer_dO = ce->dev_ptrs(ws, p.w_dO, s, p.peer_key);
    launch_dl_combine_bwd(dtype, dout, O, q.tok_of, q.kept, q.gate, q.dl, me, p.T, p.C, p.k, E, El, p.pack, p.d, peer_dO,
                          nullptr, q.dg, no_wait(s_disp), s);
    launch_sig_wait(make_sig(cm, CT::kFReadyBwdD, rb, 1, -1, nullptr, 0), s);
    prof_comm_end(cm, s);
  } else {
    launch_dl_combine_bwd(dtype, dout, O, q.tok_of, q.kept, q.gate, q.dl, me, p.T, p.C, p.k, E, El, 1, p.d, nullptr,
                          q.dO, q.dg, PeerSignal{}, s);
  }
  trace_mark(cm, s, "dl combine_bwd");
  prof_begin(cm, s);
  RowGemm d1 = dl_gemm(p, q, q.dO, w2, q.dH, p.f, p.d);
  d1.aux = q.H;
  d1.mask_in = q.mask;
  launch_expert_row_gemm(dtype, d1, false, kEpiMask, s);
  launch_expert_row_gemm(dtype, dl_gemm(p, q, q.dH, w1, q.dXe, p.d, p.f), false, kEpiNone, s);
  if (peer) {
    void* const* peer_dXs = ce->dev_ptrs(ws, p.w_dXs, s, p.peer_key);
    prof_comm_begin(cm, s);
    launch_dl_push_vsegs(dtype, q.dXe, peer_dXs, q.dl, p.V, R, E, El, p.pack, me, p.d,
                         make_sig(cm, -1, nullptr, 0, CT::kFReadyBwdC, rb, 1, kSiteCombBwd), s);
    prof_comm_end(cm, s);  // (the return rows are pushed; the wgrads overlap their arrival)
    if (cm->sched) sched_a2a_end(cm, s);
  }
  WGrad wg2{q.dO, q.H, dw2, q.dl.vcount, 1, 1, El, R, p.d, p.f};
  wg2.seg_range = q.dl.vrange;
  wg2.nseg_total = p.V;
  WGrad wg1{q.dH, q.R, dw1, q.dl.vcount, 1, 1, El, R, p.f, p.d};
  wg1.seg_range = q.dl.vrange;
  wg1.nseg_total = p.V;
  launch_expert_wgrad(dtype, wg2, s);
  launch_expert_wgrad(dtype, wg1, s);
  prof_end(cm, s, 4);
  trace_mark(cm, s, "dl dgrad x2 + wgrad x2");
  if (p.pack > 1) {  // packed experts: each replica summed its share of the rows; sum over the group
    ncclComm_t g = group_comm(cm, p.pack);
    const size_t nel = (size_t)El * p.d * p.f;
    LINA_NCCL_CHECK(ncclAllReduce(dw2, dw2, nel, nccl_dt(p), ncclSum, g, s));
    LINA_NCCL_CHECK(ncclAllReduce(dw1, dw1, nel, nccl_dt(p), ncclSum, g, s));
  }
  launch_dwg(dtype, tokens, q.probs, q.idx, q.gate, q.dg, p.T, p.d, E, p.k, q.dwg, dgate_w, s);
  if (peer) {
    const PeerSignal s_back = make_sig(cm, CT::kFReadyBwdC, rb, 1, -1, nullptr, 0, kSiteBwdEnd, rb);
    launch_sig_wait(wait_only(s_back), s);
    prof_a2a_end(cm, s);
    const PeerSignal s_back2 = no_wait(s_back);
    launch_dx(dtype, q.dXs, q.idx, q.slot, q.probs, q.gate, q.dg, gate_w, p.T, p.k, p.d, E, p.C, 1, p.C, dtokens, s,
              &s_back2, q.dl.ebase, q.dwg);
    launch_sig_wait(make_sig(cm, -1, nullptr, 0, CT::kFreeBwd, rb, 0), s);  // backward FREE
  } else {
    launch_dx(dtype, q.dXe, q.idx, q.slot, q.probs, q.gate, q.dg, gate_w, p.T, p.k, p.d, E, p.C, 1, p.C, dtokens, s,
              nullptr, q.dl.ebase, q.dwg);
  }
  trace_mark(cm, s, "dl dx");
}

}  // namespace

void moe_forward(lina_comm* cm, const Plan& p, const void* tokens, const float* gate_w,
                 const void* w1, const void* w2, void* out, void* saved, void* ws,
                 lina_route* route, cudaStream_t s) {
  trace_flush(cm);
  Ptrs q = carve(p, saved, ws);
  if (p.dropless) {  // (instrumentation flags 2 / 4 do not apply: always the full pass)
    forward_dropless(cm, p, q, tokens, gate_w, w1, w2, out, saved, route, s);
    return;
  }
  const int dtype = p.bf16 ? 1 : 0;
  const bool override_r = route && route->override_routing;
  // instrumentation (lina_profile_enable): 2 = skip collectives, 4 = collectives only
  const bool do_comm = !(cm->flags & 2), do_compute = !(cm->flags & 4);
  if (do_comm && do_compute && fused_ok(cm, p)) {
    forward_fused(cm, p, q, tokens, gate_w, w1, w2, out, saved, ws, route, s);
    return;
  }
  if (!do_compute && fused_ok(cm, p)) {  // collectives only (timing): the fused micro-ops alone
    forward_fused_movers(cm, p, q, tokens, saved, s);
    return;
  }
  const bool ce = cm->ce && p.P > 1 && do_comm;
  uint32_t seq = 0;
  if (ce) {  // every peer has pulled my previous send buffer and counts before I rewrite them
    seq = ++cm->ce->seq_fwd;
    cm->ce->prev_ce_fwd = cm->ce->last_ce_fwd;  // the previous round that used the copy engines
    cm->ce->last_ce_fwd = seq;
    for (int r = 0; r < p.P; ++r)
      if (r != cm->rank) cm->ce->wait_flag(s, CeTransport::kPulledFwdD, r, 0, cm->ce->prev_ce_fwd);
  }
  if (ce && !do_compute) {  // copy-engine collectives only (exposed-communication timing)
    cudaEvent_t e0 = cm->ev[0];
    for (int r = 0; r < p.P; ++r)
      if (r != cm->rank) cm->ce->post_flag(s, r, CeTransport::kReadyFwdD, cm->rank, 0, seq);
    LINA_CUDA_CHECK(cudaEventRecord(e0, s));
    forward_ce(cm, p, q, w1, w2, saved, ws, e0, seq, false, s);
    return;
  }
  if (!do_compute && p.P > 1) {
    cudaEvent_t* ev = cm->ev.data();
    LINA_CUDA_CHECK(cudaEventRecord(ev[0], s));
    LINA_CUDA_CHECK(cudaStreamWaitEvent(cm->hi, ev[0], 0));
    LINA_NCCL_CHECK(ncclAlltoAll(q.kept, q.recv_kept, (size_t)p.El, ncclInt32, cm->ep_disp, cm->hi));
    for (int c = 0; c < p.n; ++c) a2a_send_to_recv(p, q.D, q.R, p.d, c, cm->ep_disp, cm->hi);
    LINA_CUDA_CHECK(cudaEventRecord(ev[1], cm->hi));
    for (int c = 0; c < p.n; ++c) {
      LINA_CUDA_CHECK(cudaStreamWaitEvent(cm->hi2, ev[0], 0));
      a2a_recv_to_send(p, q.O, q.Cb, p.d, c, cm->ep_comb, cm->hi2);
    }
    LINA_CUDA_CHECK(cudaEventRecord(ev[2], cm->hi2));
    LINA_CUDA_CHECK(cudaStreamWaitEvent(s, ev[1], 0));
    LINA_CUDA_CHECK(cudaStreamWaitEvent(s, ev[2], 0));
    return;
  }
  if (override_r) {
    LINA_CUDA_CHECK(cudaMemcpyAsync(q.idx, route->idx, 4 * (size_t)p.T * p.k,
                                    cudaMemcpyDeviceToDevice, s));
    LINA_CUDA_CHECK(cudaMemcpyAsync(q.gate, route->gate, 4 * (size_t)p.T * p.k,
                                    cudaMemcpyDeviceToDevice, s));
  }
  // S1 gate, S2 route, S3 permute
  launch_gate_topk(dtype, tokens, gate_w, p.T, p.d, p.E, p.k, override_r ? 0 : 1, q.probs, q.idx,
                   q.gate, s);
  // (P = 1: the route launch also yields the chunk segments' valid rows and m-tile prefix)
  launch_route(q.idx, p.T, p.k, p.E, p.C, q.route, q.slot, route ? route->counts : nullptr,
               q.kept, q.tok_of, s, cm->route_sync, p.n, p.P == 1 ? q.vcount : nullptr,
               p.P == 1 ? q.mtp : nullptr, p.tile_rows);
  if (p.P == 1) tile_lists(p, q, s);
  launch_permute(dtype, tokens, q.tok_of, q.kept, p.k, p.d, p.E, p.C, p.n, p.Cm, q.D, s);
  if (route) {
    if (route->idx && !override_r)
      LINA_CUDA_CHECK(cudaMemcpyAsync(route->idx, q.idx, 4 * (size_t)p.T * p.k,
                                      cudaMemcpyDeviceToDevice, s));
    if (route->gate && !override_r)
      LINA_CUDA_CHECK(cudaMemcpyAsync(route->gate, q.gate, 4 * (size_t)p.T * p.k,
                                      cudaMemcpyDeviceToDevice, s));
    if (route->slot)
      LINA_CUDA_CHECK(cudaMemcpyAsync(route->slot, q.slot, 4 * (size_t)p.T * p.k,
                                      cudaMemcpyDeviceToDevice, s));
    if (route->probs)
      LINA_CUDA_CHECK(cudaMemcpyAsync(route->probs, q.probs, 4 * (size_t)p.T * p.E,
                                      cudaMemcpyDeviceToDevice, s));
  }
  if (p.P == 1) {
    // All experts local: the "all-to-all" is the identity and chunks only re-slice the GEMMs.
    trace_mark(cm, s, "P1 vcount");
    prof_begin(cm, s);
    for (int c = 0; c < p.n; ++c) {
      row_gemm(p, q.R, w1, q.H, nullptr, q.vcount, q.mtp, c, p.f, p.d, true, kEpiRelu, s, q.mask);
      trace_mark(cm, s, "P1 gemm1");
      row_gemm(p, q.H, w2, q.O, nullptr, q.vcount, q.mtp, c, p.d, p.f, true, kEpiNone, s);
      trace_mark(cm, s, "P1 gemm2");
    }
    prof_end(cm, s, 2 * p.n);
    launch_combine(dtype, q.Cb, q.idx, q.slot, q.gate, p.T, p.k, p.d, p.E, p.C, p.n, p.Cm, out, s);
    trace_mark(cm, s, "P1 combine");
    return;
  }
  // ---- P > 1: pipelined micro-ops
  cudaEvent_t* ev = cm->ev.data();
  const int n = p.n;
  cudaEvent_t e_perm = ev[0], e_cnt = ev[1], e_end = ev[2];
  if (ce) {
    for (int r = 0; r < p.P; ++r)
      if (r != cm->rank) cm->ce->post_flag(s, r, CeTransport::kReadyFwdD, cm->rank, 0, seq);
    LINA_CUDA_CHECK(cudaEventRecord(e_perm, s));
    forward_ce(cm, p, q, w1, w2, saved, ws, e_perm, seq, true, s);
    launch_combine(dtype, q.Cb, q.idx, q.slot, q.gate, p.T, p.k, p.d, p.E, p.C, p.n, p.Cm, out, s);
    return;
  }
  cudaEvent_t* e_disp = ev + 3;
  cudaEvent_t* e_gemm = ev + 3 + n;
  LINA_CUDA_CHECK(cudaEventRecord(e_perm, s));
  LINA_CUDA_CHECK(cudaStreamWaitEvent(cm->hi, e_perm, 0));
  if (do_comm) {
    LINA_NCCL_CHECK(ncclAlltoAll(q.kept, q.recv_kept, (size_t)p.El, ncclInt32, cm->ep_disp, cm->hi));
  } else {  // compute-only timing: pretend every source sent its full kept counts
    LINA_CUDA_CHECK(cudaMemcpyAsync(q.recv_kept, q.kept, 4 * (size_t)p.El, cudaMemcpyDeviceToDevice,
                                    cm->hi));
    for (int r = 1; r < p.P; ++r)
      LINA_CUDA_CHECK(cudaMemcpyAsync(q.recv_kept + (size_t)r * p.El, q.kept, 4 * (size_t)p.El,
                                      cudaMemcpyDeviceToDevice, cm->hi));
  }
  LINA_CUDA_CHECK(cudaEventRecord(e_cnt, cm->hi));
  for (int c = 0; c < n; ++c) {
    if (do_comm) a2a_send_to_recv(p, q.D, q.R, p.d, c, cm->ep_disp, cm->hi);
    LINA_CUDA_CHECK(cudaEventRecord(e_disp[c], cm->hi));
  }
  LINA_CUDA_CHECK(cudaStreamWaitEvent(s, e_cnt, 0));
  launch_vcount(q.recv_kept, p.P, p.El, p.C, n, q.vcount, s);
  launch_mtile_prefix(q.vcount, n, p.P * p.El, p.tile_rows, q.mtp, s);
  tile_lists(p, q, s);
  for (int c = 0; c < n; ++c) {
    LINA_CUDA_CHECK(cudaStreamWaitEvent(s, e_disp[c], 0));
    prof_begin(cm, s);
    row_gemm(p, q.R, w1, q.H, nullptr, q.vcount, q.mtp, c, p.f, p.d, true, kEpiRelu, s, q.mask);
    row_gemm(p, q.H, w2, q.O, nullptr, q.vcount, q.mtp, c, p.d, p.f, true, kEpiNone, s);
    prof_end(cm, s, 2);
    LINA_CUDA_CHECK(cudaEventRecord(e_gemm[c], s));
  }
  for (int c = 0; c < n; ++c) {
    LINA_CUDA_CHECK(cudaStreamWaitEvent(cm->hi2, e_gemm[c], 0));
    if (do_comm) a2a_recv_to_send(p, q.O, q.Cb, p.d, c, cm->ep_comb, cm->hi2);
  }
  LINA_CUDA_CHECK(cudaEventRecord(e_end, cm->hi2));
  LINA_CUDA_CHECK(cudaStreamWaitEvent(s, e_end, 0));
  launch_combine(dtype, q.Cb, q.idx, q.slot, q.gate, p.T, p.k, p.d, p.E, p.C, p.n, p.Cm, out, s);
}

void moe_backward(lina_comm* cm, const Plan& p, const void* saved, const void* dout,
                  const void* tokens, const float* gate_w, const void* w1, const void* w2,
                  void* dtokens, float* dgate_w, void* dw1, void* dw2, void* ws, cudaStream_t s) {
  trace_flush(cm);
  Ptrs q = carve(p, const_cast<void*>(saved), ws);
  if (p.dropless) {
    backward_dropless(cm, p, q, dout, tokens, gate_w, w1, w2, dtokens, dgate_w, dw1, dw2, ws, s);
    return;
  }
  const int dtype = p.bf16 ? 1 : 0;
  const int n = p.n;
  const bool do_comm = !(cm->flags & 2), do_compute = !(cm->flags & 4);
  if (do_comm && do_compute && fused_ok(cm, p)) {
    backward_fused(cm, p, q, dout, tokens, gate_w, w1, w2, dtokens, dgate_w, dw1, dw2, ws, s);
    return;
  }
  if (!do_compute && fused_ok(cm, p)) {
    backward_fused_movers(cm, p, q, dout, ws, s);
    return;
  }
  const bool ce = cm->ce && p.P > 1 && do_comm;
  uint32_t seq = 0;
  if (ce) {  // every peer has pulled my previous g·dY rows before combine-bwd rewrites them
    seq = ++cm->ce->seq_bwd;
    cm->ce->prev_ce_bwd = cm->ce->last_ce_bwd;
    cm->ce->last_ce_bwd = seq;
    for (int r = 0; r < p.P; ++r)
      if (r != cm->rank) cm->ce->wait_flag(s, CeTransport::kPulledBwdD, r, 0, cm->ce->prev_ce_bwd);
  }
  if (ce && !do_compute) {
    cudaEvent_t e0 = cm->ev[0];
    for (int r = 0; r < p.P; ++r)
      if (r != cm->rank) cm->ce->post_flag(s, r, CeTransport::kReadyBwdD, cm->rank, 0, seq);
    LINA_CUDA_CHECK(cudaEventRecord(e0, s));
    backward_ce(cm, p, q, w1, w2, dw1, dw2, ws, e0, seq, dtype, false, s);
    return;
  }
  if (!do_compute && p.P > 1) {  // collectives-only timing
    cudaEvent_t* ev = cm->ev.data();
    LINA_CUDA_CHECK(cudaEventRecord(ev[0], s));
    LINA_CUDA_CHECK(cudaStreamWaitEvent(cm->hi, ev[0], 0));
    LINA_CUDA_CHECK(cudaStreamWaitEvent(cm->hi2, ev[0], 0));
    for (int c = 0; c < n; ++c) a2a_send_to_recv(p, q.dS, q.dO, p.d, c, cm->ep_disp, cm->hi);
    for (int c = 0; c < n; ++c) a2a_recv_to_send(p, q.dXe, q.dXs, p.d, c, cm->ep_comb, cm->hi2);
    LINA_CUDA_CHECK(cudaEventRecord(ev[1], cm->hi));
    LINA_CUDA_CHECK(cudaEventRecord(ev[2], cm->hi2));
    LINA_CUDA_CHECK(cudaStreamWaitEvent(s, ev[1], 0));
    LINA_CUDA_CHECK(cudaStreamWaitEvent(s, ev[2], 0));
    return;
  }
  // (a) combine backward: dg and g·dY rows into the send layout
  launch_combine_bwd(dtype, dout, q.Cb, q.tok_of, q.kept, q.gate, p.T, p.k, p.d, p.E, p.C, n, p.Cm, q.dS,
                     q.dg, s);
  // the scheduler stops admitting allreduce micro-ops: all-to-all is imminent
  if (cm->sched) sched_a2a_imminent(cm, s);
  WGrad wg2{q.dO, q.H, dw2, q.vcount, n, p.P, p.El, p.Cm, p.d, p.f};
  WGrad wg1{q.dH, q.R, dw1, q.vcount, n, p.P, p.El, p.Cm, p.f, p.d};
  bool dwg_done = false;
  if (ce) {
    for (int r = 0; r < p.P; ++r)
      if (r != cm->rank) cm->ce->post_flag(s, r, CeTransport::kReadyBwdD, cm->rank, 0, seq);
    cudaEvent_t e_cb = cm->ev[0];
    LINA_CUDA_CHECK(cudaEventRecord(e_cb, s));
    backward_ce(cm, p, q, w1, w2, dw1, dw2, ws, e_cb, seq, dtype, true, s);
  } else if (p.P == 1) {
    prof_begin(cm, s);
    for (int c = 0; c < n; ++c) {
      row_gemm(p, q.dO, w2, q.dH, q.H, q.vcount, q.mtp, c, p.f, p.d, false, kEpiMask, s, nullptr, q.mask);
      row_gemm(p, q.dH, w1, q.dXe, nullptr, q.vcount, q.mtp, c, p.d, p.f, false, kEpiNone, s);
    }
    launch_expert_wgrad(dtype, wg2, s);
    launch_expert_wgrad(dtype, wg1, s);
    prof_end(cm, s, 2 * n + 2);
  } else {
    cudaEvent_t* ev = cm->ev.data();
    cudaEvent_t e_cb = ev[0], e_end = ev[1], e_wg = ev[2];
    cudaEvent_t* e_disp = ev + 3;
    cudaEvent_t* e_gemm = ev + 3 + n;
    LINA_CUDA_CHECK(cudaEventRecord(e_cb, s));
    LINA_CUDA_CHECK(cudaStreamWaitEvent(cm->hi, e_cb, 0));
    if (cm->sched) sched_a2a_begin(cm, cm->hi);
    for (int c = 0; c < n; ++c) {
      if (do_comm) a2a_send_to_recv(p, q.dS, q.dO, p.d, c, cm->ep_disp, cm->hi);
      LINA_CUDA_CHECK(cudaEventRecord(e_disp[c], cm->hi));
    }
    for (int c = 0; c < n; ++c) {
      LINA_CUDA_CHECK(cudaStreamWaitEvent(s, e_disp[c], 0));
      prof_begin(cm, s);
      row_gemm(p, q.dO, w2, q.dH, q.H, q.vcount, q.mtp, c, p.f, p.d, false, kEpiMask, s, nullptr, q.mask);
      row_gemm(p, q.dH, w1, q.dXe, nullptr, q.vcount, q.mtp, c, p.d, p.f, false, kEpiNone, s);
      prof_end(cm, s, 2);
      LINA_CUDA_CHECK(cudaEventRecord(e_gemm[c], s));
    }
    for (int c = 0; c < n; ++c) {
      LINA_CUDA_CHECK(cudaStreamWaitEvent(cm->hi2, e_gemm[c], 0));
      if (do_comm) a2a_recv_to_send(p, q.dXe, q.dXs, p.d, c, cm->ep_comb, cm->hi2);
    }
    LINA_CUDA_CHECK(cudaEventRecord(e_end, cm->hi2));
    if (cm->sched) sched_a2a_end(cm, cm->hi2);
    // weight gradients after every chunk: off the critical path, overlap the last combine a2a
    prof_begin(cm, s);
    launch_expert_wgrad(dtype, wg2, s);
    launch_expert_wgrad(dtype, wg1, s);
    prof_end(cm, s, 2);
    // (e)+(f) dWg needs only this rank's dg: it overlaps the last combine all-to-all
    launch_dwg(dtype, tokens, q.probs, q.idx, q.gate, q.dg, p.T, p.d, p.E, p.k, q.dwg, dgate_w, s);
    LINA_CUDA_CHECK(cudaEventRecord(e_wg, s));
    LINA_CUDA_CHECK(cudaStreamWaitEvent(s, e_end, 0));
    dwg_done = true;
  }
  if (!dwg_done)
    launch_dwg(dtype, tokens, q.probs, q.idx, q.gate, q.dg, p.T, p.d, p.E, p.k, q.dwg, dgate_w, s);
  // (e)+(f): gate backward + gather-sum dX
  launch_dx(dtype, q.dXs, q.idx, q.slot, q.probs, q.gate, q.dg, gate_w, p.T, p.k, p.d, p.E, p.C, n, p.Cm,
            dtokens, s, nullptr, nullptr, q.dwg);
}

}  // namespace lina
