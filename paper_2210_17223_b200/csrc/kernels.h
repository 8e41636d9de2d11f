// Internal kernel launchers of the Lina B200 library.  All launches are
// asynchronous on the given stream; they throw lina::CudaError on launch failure.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include <vector>

#include "signal.h"

namespace lina {

enum { kEpiNone = 0, kEpiRelu = 1, kEpiMask = 2 };

// Row-grouped expert GEMM over the segments of one chunk (see gemm_simt.cu).
struct RowGemm {
  const void* A;       // [nseg_total][Cm][K]
  const void* B;       // [El][N][K] (K-major) or [El][K][N] (MN-major)
  void* D;             // [nseg_total][Cm][N]
  const void* aux;     // [nseg_total][Cm][N] (kEpiMask: keep where aux > 0)
  const int* vcount;   // [nseg_total] valid rows per segment
  const int* mtp;      // [nseg+1] prefix of valid 128-row blocks over this launch's segments
  int seg0, nseg, El, Cm, N, K;
  const int* seg_expert = nullptr;  // [El] weight index of local slot (seg % El); NULL = identity
  int B_experts = 0;                // expert matrices in B (0 = El)
  uint64_t* mask_out = nullptr;       // tcgen05 ReLU epilogue: ReLU' bits [nseg_total][N/64][Cm]
  const uint64_t* mask_in = nullptr;  // tcgen05 mask epilogue: those bits (aux unused)
  const PeerSignal* sig = nullptr;    // tcgen05: wait before the first A load, post after the last store
  int tile_rows = 256;                // tcgen05 M tile (256: CTA pairs, 128: single CTAs); = mtp's rows
  // tail split (tile_rows 256, tcgen05): mtp counts each segment's 256-row tiles except a
  // last one holding <= 128 rows, which a second launch computes as a 128-row single-CTA
  // tile (mtp_tail: prefix of those [nseg+1]; row_base[global segment] = its first row) —
  // a 129th..256th row costs a full 256-row MMA, a <= 128-row tail only half of one
  const int* mtp_tail = nullptr;
  const int* row_base = nullptr;
  // half tails (tile_rows 256, tcgen05, no tail split): a segment's last m-tile holding
  // <= 128 valid rows runs in the same launch as an M = 128 cta_group::2 tile (64 rows per
  // CTA of the pair) — half the MMA time of the 256-row tile, no second launch
  int half_tails = 0;
  // split dispatch (tcgen05, n = 1): sig.wait is per source — the TMA producer waits for
  // source s's slot before its first A load of a segment of s, and tiles are walked from
  // source src_me upwards (the order the sources' rows arrive in, permute.cu)
  int src_wait = 0, src_P = 1, src_me = 0;
};

// Weight-gradient GEMM: D[El][M][N] = Σ_{c,s} Σ_{r < v} A[seg][r][:]ᵀ B[seg][r][:].
struct WGrad {
  const void* A;       // [nseg_total][Cm][M]
  const void* B;       // [nseg_total][Cm][N]
  void* D;             // [El][M][N]
  const int* vcount;
  int nchunks, P, El, Cm, M, N;
  // dropless layout: expert el sums segments [seg_range[2el], seg_range[2el+1]) of
  // nseg_total (instead of segments (c*P + s)*El + el)
  const int* seg_range = nullptr;
  int nseg_total = 0;
};

// sig (fused transport): block 0 posts sig at kernel start (the FREE of this round).
void launch_gate_topk(int dtype, const void* X, const float* Wg, int T, int d, int E, int k,
                      int write_routing, float* probs, int* idx, float* gate, cudaStream_t s,
                      const PeerSignal* sig = nullptr);

// tcgen05 gate (gate_tc.cu): logits on the tensor cores, softmax / top-k in the epilogue.
bool gate_tc_supported(int d, int E, int k);
void launch_gate_tc(const void* X, const float* Wg, int T, int d, int E, int k, int write_routing, float* probs,
                    int* idx, float* gate, const PeerSignal& sig, cudaStream_t s);

size_t route_scratch_ints(int T, int k, int E);
// sync: zeroed device words (route_sync_words(), comm-owned) -> one fused launch;
// NULL -> the three-launch count / scan / assign path.  vcount/mtp (P = 1 only): also
// the chunk segments' valid rows [n][E] and m-tile prefix [n][E+1] of `tile_rows` rows.
size_t route_sync_words();
void launch_route(const int* idx, int T, int k, int E, int C, int* scratch, int* slot, int* counts,
                  int* kept, int* tok_of, cudaStream_t s, unsigned int* sync = nullptr, int n_chunks = 1,
                  int* vcount = nullptr, int* mtp = nullptr, int tile_rows = 256);
// vcount[(c*P + s)*El + el] = clamp(recv_kept[s*El + el] - b_c, 0, Cc)
// A 1-CTA kernel that waits for sig's flags, then publishes sig.post and bumps sig.bump
// (each part optional).  Callers pass no_wait()-style signals to the consumer kernel.
void launch_sig_wait(const PeerSignal& sig, cudaStream_t s);
// Row blocks to peers over NVLink: block b copies rows [src_row[b], +nrows[b]) of `src`
// to peer_dst[b] + dst_row[b] (rows of d elements); the last CTA posts sig.
void launch_push_blocks(int dtype, const void* src, void* const* peer_dst, const int* blocks /*[P][3]*/, int P,
                        int d, int max_rows, const PeerSignal& sig, cudaStream_t s);
// sig: every CTA first waits for the peers' counts (READY of the dispatch)
void launch_vcount(const int* recv_kept, int P, int El, int C, int n, int* vcount, cudaStream_t s,
                   const PeerSignal* sig = nullptr);

// Rows past the first 64-row boundary after a segment's kept rows are not written (see
// permute.cu kRowSkip); kept[e] = this rank's kept count of expert e.
void launch_permute(int dtype, const void* X, const int* tok_of, const int* kept, int k, int d, int E, int C,
                    int n, int Cm, void* Send, cudaStream_t s);
// sig: block 0 posts sig.post (FREE of the backward buffers) at start; every CTA waits
// sig.wait (the returned expert outputs) before reading Recv.
// ebase (dropless layout): row of (t, j) = ebase[idx] + slot instead of the send-layout row.
void launch_combine(int dtype, const void* Recv, const int* idx, const int* slot, const float* gate,
                    int T, int k, int d, int E, int C, int n, int Cm, void* Y, cudaStream_t s,
                    const PeerSignal* sig = nullptr, const int* ebase = nullptr);
void launch_combine_bwd(int dtype, const void* dY, const void* Recv, const int* tok_of, const int* kept,
                        const float* gate, int T, int k, int d, int E, int C, int n, int Cm,
                        void* dSend, float* dg, cudaStream_t s);
// dX (gather-sum + dL·Wgᵀ) and dWg (Xᵀ dL) with dL recomputed from the forward routing.
// tc_scratch: the dWg scratch of the same backward (its launch_dwg ran first): the
// tensor-core path reads the dL split from it; NULL = the CUDA-core kernel.
void launch_dx(int dtype, const void* dXe, const int* idx, const int* slot, const float* probs,
               const float* gate, const float* dg, const float* Wg, int T, int k, int d, int E, int C,
               int n, int Cm, void* dX, cudaStream_t s, const PeerSignal* sig = nullptr,
               const int* ebase = nullptr, const void* tc_scratch = nullptr);
// tensor-core gate backward (gate_bwd_tc.cu)
bool gate_bwd_tc_supported(int dtype, int d, int E, int k);
size_t gate_bwd_tc_scratch_bytes(int T, int d, int E);
void launch_dwg_tc(const void* X, const float* probs, const int* idx, const float* gate, const float* dg, int T,
                   int d, int E, int k, void* scratch, float* dWg, cudaStream_t s);
void launch_dx_tc(const void* dXe, const int* idx, const int* slot, const float* Wg, int T, int k, int d, int E,
                  int C, int n, int Cm, const int* ebase, void* dX, const void* scratch, const PeerSignal& sig,
                  cudaStream_t s);
void launch_dwg_reduce(const float* part, int nparts, int dE, float* dWg, cudaStream_t s);
size_t dwg_scratch_floats(int T, int d, int E);
void launch_dwg(int dtype, const void* X, const float* probs, const int* idx, const float* gate,
                const float* dg, int T, int d, int E, int k, float* scratch, float* dWg, cudaStream_t s);

// CTAs per tensor-core tile (cta_group::2 pairs -> 256-row tiles) of the wgrad and the
// default row GEMM; row GEMMs may also run 128-row single-CTA tiles (RowGemm::tile_rows).
constexpr int kTcCtaGroup = 2;
int tc_tile_rows();
// SMs the persistent GEMM grid leaves free for concurrently running NCCL kernels.
void tc_set_reserved_sms(int n);
// The dynamic tile-schedule counter of the calling communicator (NULL: static schedule).
void tc_set_tile_counter(unsigned int* ctr);
// mtp[c][i] = Σ_{i' < i} ceil(vcount[c*nseg + i'] / rows), i in [0, nseg]  (tcgen05 tile lists)
void launch_mtile_prefix(const int* vcount, int n, int nseg, int rows, int* mtp, cudaStream_t s);
// the tail-split lists: mtp[c][nseg+1] (256-row tiles, a last tile only when it holds > 128
// rows), mtp_tail[c][nseg+1] (one 128-row tile per segment whose remainder is 1..128 rows),
// rbase[c][nseg] (that tile's first row)
void launch_mtile_split(const int* vcount, int n, int nseg, int* mtp, int* mtp_tail, int* rbase, cudaStream_t s);
bool tc_row_supported(const RowGemm& g);
bool tc_wgrad_supported(const WGrad& g);
void launch_row_gemm_tc(const RowGemm& g, bool b_kmajor, int epi, cudaStream_t s);
void launch_wgrad_tc(const WGrad& g, cudaStream_t s);

// fused dispatch over NVLink peer stores (permute.cu): rows go straight into the owners'
// receive buffers (peer_rows[o]) and the counts into their recv_kept (peer_counts[o]).
// sig: every CTA waits for the peers' FREE, block 0 also stores this rank's counts into
// the owners' recv_kept (peer_counts[o]), and the last CTA posts READY.
// [c0, c0 + nc): the micro-op chunks this launch moves (counts are stored with chunk 0).
void launch_permute_peer(int dtype, const void* X, const int* tok_of, const int* kept, int k, int d, int E,
                         int C, int c0, int nc, int Cm, int El, int P, int me, void* const* peer_rows,
                         void* const* peer_counts, const PeerSignal& sig, cudaStream_t s);
void launch_combine_bwd_peer(int dtype, const void* dY, const void* Recv, const int* tok_of, const int* kept,
                             const float* gate, int T, int k, int d, int E, int C, int c0, int nc, int Cm, int El,
                             int P, int me, void* const* peer_rows, float* dg, const PeerSignal& sig,
                             cudaStream_t s);
// Split dispatch (n = 1; permute.cu split_rows_kernel): the owner blocks j0 .. j0+nj-1 in
// the order owner(j) = (me - j) mod P (j = 0: this rank's own block), grid CTAs (0 = one
// pass), the last CTA done with block j > 0 posts sig's READY to owner(j) (done[j] = its
// zeroed counter); sig.wait (if set) is awaited by every CTA first.  The combine-backward
// variant also writes dg of its rows (dg zeroed by the caller).
void launch_dispatch_counts(const int* kept, int P, int El, int me, void* const* peer_counts,
                            const PeerSignal& free_sig, const PeerSignal& count_sig, cudaStream_t s);
void launch_permute_split(int dtype, const void* X, const int* tok_of, const int* kept, int k, int d, int E, int C,
                          int Cm, int El, int P, int me, void* const* peer_rows, int j0, int nj, int grid,
                          const PeerSignal& sig, unsigned int* done, cudaStream_t s);
void launch_combine_bwd_split(int dtype, const void* dY, const void* Recv, const int* tok_of, const int* kept,
                              const float* gate, int k, int d, int E, int C, int Cm, int El, int P, int me,
                              void* const* peer_rows, float* dg, int j0, int nj, int grid, const PeerSignal& sig,
                              unsigned int* done, cudaStream_t s);
// Collectives-only timing (movers.cu): the valid rows of micro-op c's segments of a
// receive-layout buffer to each owner's send-layout buffer (peer_send_layout[s]), as the
// peer-storing GEMM epilogue moves them; the last CTA posts sig (READY of micro-op c).
void launch_push_segments(int dtype, const void* recv_layout, void* const* peer_send_layout, const int* vcount,
                          int c, int P, int El, int E, int Cm, int me, int d, const PeerSignal& sig, cudaStream_t s);
// Dropless training (dropless.cu; §8(f) row 4): tables computed on the device from the
// exchanged per-expert counts allc [P][E] (identical on every rank).
struct DlTables {
  int* dbase;      // [E]   first row of this rank's block for expert e at its owner (dispatch target)
  int* ebase;      // [E]   first row of this rank's expert-e rows where the combine reads them
  int* soff;       // [P][E] compact source offsets: Σ_{e'<e} allc[s][e']
  int* src_total;  // [P]   rows each source sends in total (= T_s·k)
  int* vcount;     // [V]   valid rows of each virtual segment of this rank (0 past the used ones)
  int* vexp;       // [V]   local expert (weight index) of the segment
  int* vsrc;       // [V]   source rank of the segment's rows
  int* vq0;        // [V]   first slot (within the source's expert block) of the segment
  int* mtp;        // [V+1] m-tile prefix (one tile per used segment; with the tail split: > 128 rows)
  int* mtpt;       // [V+1] tail-split prefix: segments holding 1..128 rows
  int* vrange;     // [E_l][2] segment range of each local expert (wgrad)
};
void launch_dl_counts(const int* kept, int* const* peer_allc, int P, int me, int E, const PeerSignal& sig,
                      cudaStream_t s);
void launch_dl_layout(const int* allc, int P, int E, int El, int m, int me, int R, int V, int split, const DlTables& t,
                      cudaStream_t s);
// peer_dst: device array [P] of the owners' buffers (fused transport), or NULL and local_dst.
// El = experts hosted per rank, m = packing factor (owner of my rows of e: (e/El)*m + me%m).
void launch_dl_permute(int dtype, const void* X, const int* tok_of, const int* kept, const DlTables& t, int me,
                       int T, int C, int k, int E, int El, int m, int d, void* const* peer_dst, void* local_dst,
                       const PeerSignal& sig, cudaStream_t s);
void launch_dl_combine_bwd(int dtype, const void* dY, const void* O, const int* tok_of, const int* kept,
                           const float* gate, const DlTables& t, int me, int T, int C, int k, int E, int El, int m, int d,
                           void* const* peer_dst, void* local_dst, float* dg, const PeerSignal& sig, cudaStream_t s);
void launch_dl_push_vsegs(int dtype, const void* src, void* const* peer, const DlTables& t, int V, int R, int E,
                          int El, int m, int me, int d, const PeerSignal& sig, cudaStream_t s);
// Output tiles of a row GEMM stored through per-owner tensor maps (peer memory):
// segment (c, s, el) of the receive layout goes to map s at segment c*E + me*El + el.
struct PeerStore {
  const void* host_maps = nullptr;  // host array [P] of CUtensorMap (tc_peer_dmaps), copied into the launch
  char* const* bases = nullptr;     // host array [P]: the same buffers (mapped here)
  int P = 0, me = 0, E = 0;
};
void launch_row_gemm_tc_peer(const RowGemm& g, bool b_kmajor, int epi, const PeerStore& ps, cudaStream_t s);
// Host bytes of the P tensor maps of `bases[r]` viewed as [nseg][Cm][N] bf16 (box 64 x 32).
std::vector<unsigned char> tc_peer_dmaps(const std::vector<char*>& bases, int N, int Cm, int nseg);

// inference replica routing (infer_route.cu); tab = r[E] | rdev[E][N] | send_off[N][E] | cnt[E]
void launch_infer_permute(int dtype, const void* X, const int* idx, const int* slot, const int* tab,
                          int T, int k, int d, int E, int N, int s, void* Send, int* arow,
                          cudaStream_t st);
void launch_combine_rows(int dtype, const void* Back, const int* arow, const float* gate, int T, int k,
                         int d, void* Y, cudaStream_t st);
// source-major [P][mpd][rows] <-> expert-major [mpd][Cm] rows (nrecv[P][mpd] device table)
void launch_regroup(int dtype, const void* src, void* dst, const int* nrecv, int P, int mpd, int Cm, int d,
                    int max_rows, bool to_expert_major, cudaStream_t st);

void launch_row_gemm_simt(int dtype, const RowGemm& p, bool b_kmajor, int epi, cudaStream_t s);
void launch_wgrad_simt(int dtype, const WGrad& p, cudaStream_t s);

}  // namespace lina
