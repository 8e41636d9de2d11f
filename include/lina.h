/*
 * lina.h — C ABI of the B200-native Lina expert-parallel MoE layer.
 *
 * What is computed (PAPER.md = arXiv 2210.17223, "Accelerating Distributed MoE
 * Training and Inference with Lina"; P:n = PAPER.md line n):
 *   An MoE layer "consists of multiple FFNs each serving as an expert, and a
 *   gating network ... Every expert is a fully-connected two-layer network using
 *   ReLU ... The gating network takes in the embedding vector of each token and
 *   multiplies them with its trainable matrix. Based on the results, it
 *   dispatches the token to a small number of experts ... The final output of
 *   the MoE layer is the weighted sum of outputs from the selected expert(s)"
 *   (§2.1).  With expert parallelism "an all-to-all communication is then
 *   needed to send tokens to their experts selected by the gating network, and
 *   another all-to-all is needed to send tokens back".
 *   Lina partitions the all-to-all into micro-ops along the token dimension and
 *   pipelines the expert FFN behind them (§4.2; §6.1),
 *   gives all-to-all strict priority over the gradient allreduce, whose tensors
 *   are split into equal micro-ops (§3, §4.2, §6.1),
 *   and in inference replicates popular experts by Eq. (1) with first-fit-
 *   decreasing packing (§5.2) and an unequal-split all-to-all,
 *   planning from a sample-path popularity estimate before gating and checking it
 *   against the gate's top-2k after (two-phase scheduling).
 *   Readings where the paper is silent (capacity, drop order, gate
 *   normalisation, tie-breaks, rounding points, sample paths) are R1-R22 in DESIGN.md §3.
 *
 * Conventions for every entry point:
 *   - Every function returns lina_status; nothing throws across the ABI.  On a
 *     non-OK status, lina_last_error() returns a thread-local message; for
 *     LINA_ERR_INVALID_ARGUMENT it lists EVERY violated invariant.
 *   - Pointers named *device* / all tensor arguments of lina_moe_* are CUDA
 *     device pointers on the communicator's device, caller-owned, row-major,
 *     contiguous, 16-byte aligned.  Host arrays are named host_* or documented.
 *   - All device work is enqueued on the caller's `stream` (a cudaStream_t
 *     passed as void*; NULL = legacy default stream).  Internal streams fork
 *     from and join back to `stream` with events; results are valid when
 *     `stream` reaches that point.  Pointers must stay live until then.  The
 *     calls never synchronise the host, except lina_moe_infer_forward (the
 *     unequal all-to-all needs host-visible counts).
 *   - lina_moe_forward / lina_moe_backward may be captured in a CUDA graph
 *     (after one eager call on the same buffers, which sets up the peer
 *     mappings): the cross-rank ordering of the fused all-to-all keeps its
 *     rounds in device memory, so every replay is a complete step.  All ranks
 *     must issue the same sequence of calls.
 *   - Training all-to-all transport (environment, read at lina_comm_init):
 *     LINA_TRANSPORT=fused (default: peer stores from the permute / combine-
 *     backward kernels and the GEMM epilogues over NVLink, in-kernel flags),
 *     ce (copy engines) or nccl (ncclAlltoAll micro-ops).  LINA_TRACE=1 prints a
 *     per-phase device-time trace per rank at lina_comm_destroy.  LINA_PDL=0 turns
 *     off programmatic dependent launch; LINA_TILE_ROWS=128|256 forces the expert
 *     row-GEMM tile height (default: 128 when segments average <= 96 rows).
 *   - The library never allocates caller-visible memory in forward/backward:
 *     scratch and saved state are caller-allocated, sized by
 *     lina_moe_workspace_size().
 *   - One lina_comm per rank (process/GPU).  Calls on one lina_comm are not
 *     reentrant, and the work of its layer calls must be ordered on one stream
 *     (its expert GEMMs draw their tiles from one self-resetting device counter
 *     owned by the comm: the dynamic tile schedule; LINA_GEMM_DYN=0 at
 *     lina_comm_init selects the static schedule, which has no such state).
 *     There is NO CPU fallback: on a machine without an sm_100 GPU
 *     lina_comm_init fails with LINA_ERR_UNSUPPORTED.
 */
#ifndef LINA_H_
#define LINA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LINA_OK = 0,
  LINA_ERR_INVALID_ARGUMENT = 1, /* descriptor / pointer invariant violated (all listed)      */
  LINA_ERR_UNSUPPORTED = 2,      /* valid but not implemented here (e.g. no sm_100 device)     */
  LINA_ERR_INFEASIBLE_PLAN = 3,  /* E > N * max_per_device, or a replica cannot be placed      */
  LINA_ERR_CUDA = 4,             /* a CUDA runtime/driver call failed (message has the name)   */
  LINA_ERR_NCCL = 5,             /* an NCCL call failed or the communicator reported an error  */
  LINA_ERR_WORKSPACE = 6         /* workspace/saved buffer smaller than lina_moe_workspace_size */
} lina_status;

typedef enum {
  LINA_F32 = 0,  /* fp32 tokens/weights/outputs; expert GEMMs on CUDA cores (no TF32)        */
  LINA_BF16 = 1  /* bf16 tokens/weights/outputs; expert GEMMs on tcgen05 tensor cores, fp32 acc */
} lina_dtype;

typedef enum {
  /* Non-expert allreduce micro-ops are issued as soon as their gradient is
   * ready, whole tensors, on the low-priority stream — concurrent with the
   * all-to-all and fair-sharing the links (the paper's DeepSpeed baseline,
   * P:64, fig:schedule_baseline P:283). */
  LINA_SCHED_BASELINE = 0,
  /* Lina: each gradient is split into equal partition_bytes micro-ops (never
   * mixing gradients); a micro-op is launched only while no
   * all-to-all micro-op is queued or in flight; launching stops
   * once the combine backward starts, "since this implies all-to-all is
   * imminent". */
  LINA_SCHED_LINA = 1,
  /* Ablation (fig:schedule_naive P:289): strict priority without
   * partitioning — a ready gradient is issued WHOLE, and only while no all-to-all
   * is queued or in flight (the LINA admission rule); once launched it cannot be
   * preempted (R23). */
  LINA_SCHED_NAIVE = 2,
  /* Ablation: "blindly defer allreduce until an even number of
   * all-to-all finish" — a ready gradient waits only for the backward all-to-all
   * phase in flight (dispatch + combine, two all-to-alls) to complete, then is
   * issued WHOLE, without regard to the next all-to-all (R23). */
  LINA_SCHED_DEFER = 3
} lina_policy;

typedef void* lina_stream; /* cudaStream_t */
typedef struct lina_comm lina_comm;

/* ------------------------------------------------------------------------ */
/* Errors, version                                                           */
/* ------------------------------------------------------------------------ */

/* Thread-local message for the last non-OK status on this thread ("" if none). */
const char* lina_last_error(void);
/* Library version and build arch string, e.g. "lina 0.1 sm_100a". */
const char* lina_version(void);

/* ------------------------------------------------------------------------ */
/* Communicator: one per rank.  Expert-parallel (EP) and data-parallel (DP)   */
/* NCCL communicators over the same world (the paper's separate EP and DP    */
/* process groups, each on its own CUDA stream), a high-priority stream */
/* for all-to-all micro-ops and a low-priority stream for allreduce micro-ops.*/
/* ------------------------------------------------------------------------ */

/* Rank 0 creates an NCCL unique id (128 bytes, host memory) that the caller
 * broadcasts to the other ranks (e.g. through its torch process group). */
lina_status lina_get_unique_id(unsigned char host_id[128]);

/* world >= 1, 0 <= rank < world, cuda_device = local GPU index.  host_id may
 * be NULL only when world == 1 (no NCCL is created: the P=1 layer needs no
 * collective).  nccl_max_ctas > 0 caps the SMs each NCCL kernel may take
 * (ncclConfig_t.maxCTAs) so the expert GEMM keeps the rest; 0 = NCCL default.
 * Errors: INVALID_ARGUMENT, UNSUPPORTED (device is not sm_100), CUDA, NCCL. */
lina_status lina_comm_init(int world, int rank, int cuda_device, const unsigned char* host_id,
                           int nccl_max_ctas, lina_comm** out);
/* A communicator without NCCL: the ranks' bootstrap exchanges (the peer-memory handles,
 * the inference counts, barriers) go through a caller-supplied HOST allgather —
 * fn(send, recv, bytes, ctx) gathers `bytes` from every rank into recv [world][bytes] in
 * rank order and returns 0 on success (e.g. a torch gloo all_gather).  All-to-alls use the
 * fused transport (NVLink peer stores, in-kernel flags); what needs an NCCL collective is
 * UNSUPPORTED on it: the allreduce scheduler (lina_allreduce_submit with world > 1), the
 * nccl / ce transports and expert packing's group sum.  Several ranks may share one GPU
 * (NCCL refuses that): their kernels time-slice and the in-kernel flag waits still order
 * them — slow, but it lets one GPU run the multi-rank data path (tests).  fn is called
 * from the calling thread only, inside lina calls.
 * Errors: INVALID_ARGUMENT, UNSUPPORTED (device is not sm_100), CUDA. */
typedef int (*lina_host_allgather_fn)(const void* send, void* recv, size_t bytes, void* ctx);
lina_status lina_comm_init_host(int world, int rank, int cuda_device, lina_host_allgather_fn fn, void* ctx,
                                lina_comm** out);
/* Waits for the scheduler thread, destroys comms/streams/events.  NULL is a no-op. */
lina_status lina_comm_destroy(lina_comm* comm);
/* Surfaces asynchronous NCCL/CUDA errors (ncclCommGetAsyncError, cudaPeekAtLastError). */
lina_status lina_comm_check(lina_comm* comm);
/* rank / world of a communicator. */
lina_status lina_comm_info(const lina_comm* comm, int* rank, int* world);

/* ------------------------------------------------------------------------ */
/* Placement / replication tables (paper D3: expert -> device mapping,        */
/* replica list and per-replica token split; Eq. (1)).  */
/* All arrays are HOST memory owned by the caller.                            */
/* ------------------------------------------------------------------------ */
typedef struct {
  int32_t num_experts;    /* E                                                        */
  int32_t num_devices;    /* N (= world)                                              */
  int32_t max_per_device; /* at most this many experts hosted per device (4)   */
  int32_t max_replicas;   /* row pitch of replica_device; >= max r_e (N is always enough) */
  int32_t* replicas;      /* [E]                 r_e >= 1                              */
  int32_t* replica_device;/* [E][max_replicas]   device ids ascending, -1 padded       */
  int32_t* hosted;        /* [N][max_per_device] expert ids ascending, -1 padded       */
} lina_placement;

/* Eq. (1) n_e = N * popularity[e]; r_e = max(1, round-half-up(n_e)) capped at N,
 * trimmed largest-first while sum r_e > N*max_per_device; replicas (size n_e/r_e
 * device-loads) packed first-fit-decreasing into devices of capacity 1.0
 * (P:478); an item that fits nowhere goes to the least-loaded eligible device
 * (lowest id), the deterministic stand-in for "randomly assigned".
 * popularity: host [E], >= 0 (need not sum to 1).  `out` arrays caller-allocated
 * with the pitches above.  Errors: INVALID_ARGUMENT, INFEASIBLE_PLAN
 * (E > N*max_per_device).  Pure host function, no device needed. */
lina_status lina_placement_compute(const double* host_popularity, int32_t num_experts,
                                   int32_t num_devices, int32_t max_per_device,
                                   lina_placement* out);

/* Tokens a source rank sends to each replica of one expert (R14: contiguous
 * blocks in slot order whose sizes differ by <= 1; block q goes to replica
 * (q + source_rank) mod r_e).  host_out[r_e]. */
lina_status lina_replica_split(int32_t count, int32_t replicas, int32_t source_rank,
                               int32_t* host_out);

/* ------------------------------------------------------------------------ */
/* Popularity estimation and two-phase scheduling (§5.2;  */
/* paper D4: per-layer popularity distributions kept in host DRAM).    */
/* Pure host functions, no device needed.  Readings R19-R22:   */
/*  - a sample path of length l ending at layer i = the token's selected      */
/*    expert SETS at layers i-l+1..i (l >= 1);                                */
/*  - Psi_j^{m}(e) = tokens of path j selecting e in layer m / (k * |j|);     */
/*  - an unseen path backs off to its suffixes l-1..1, then layer m's         */
/*    marginal;                                                               */
/*  - top-k ties go to the lower expert id.                                   */
/* Layers are 0-indexed.                                                      */
/* ------------------------------------------------------------------------ */
typedef struct lina_pop_profile lina_pop_profile;  /* lina_popprof_add must not overlap
                                                      any other call on the same profile;
                                                      concurrent estimates are safe (read only) */

/* An empty profile.  num_layers >= 2, num_experts >= 1, 1 <= k <= num_experts,
 * 1 <= path_len < num_layers.  Errors: INVALID_ARGUMENT (all violations listed). */
lina_status lina_popprof_create(int32_t num_layers, int32_t num_experts, int32_t k, int32_t path_len,
                                lina_pop_profile** out);
/* Frees the profile.  NULL is a no-op. */
lina_status lina_popprof_destroy(lina_pop_profile* prof);
/* "collect the expert selection results of all tokens" and group them by
 * sample path: host_sel [num_tokens][num_layers][k] int32 expert ids
 * (host memory, read only during the call).  Counts accumulate over calls.
 * Errors: INVALID_ARGUMENT (NULL, num_tokens < 0, an id outside [0, E), or a token
 * selecting one expert twice in a layer); the profile is unchanged on error. */
lina_status lina_popprof_add(lina_pop_profile* prof, const int32_t* host_sel, int64_t num_tokens);
/* Phase-one estimate of layer `layer`'s expert popularity for a batch, before any of
 * its computation: each token t takes the top-k experts of its path's
 * Psi and contributes their probabilities P_j(e); host_popularity[e] =
 * (sum_t P_{j(t)}(e)) / num_tokens in fp64, summed in token order (Eq. (1)'s overall
 * popularity).  host_history [num_tokens][path_len][k] = each token's
 * selections at layers layer-path_len .. layer-1.  host_topk [num_tokens][k] (may be
 * NULL) receives each token's chosen experts, -1 for a token with no distribution.
 * A batch with num_tokens == 0 yields all zeros.  Errors: INVALID_ARGUMENT (layer <
 * path_len or >= num_layers, bad ids, NULL). */
lina_status lina_popprof_estimate(const lina_pop_profile* prof, int32_t layer, const int32_t* host_history,
                                  int64_t num_tokens, double* host_popularity, int32_t* host_topk);
/* Persist a profile built offline from training traces ("In the profiling stage",
 * P:428) for use at inference: a little-endian binary file (magic "LINAPOP1", the
 * shape, the layer marginals and every sample-path entry); load returns a new profile
 * (free it with lina_popprof_destroy) whose estimates equal the saved one's.  Errors:
 * INVALID_ARGUMENT for a NULL argument or an unwritable, unreadable or malformed file
 * (the message says which).  Host only. */
lina_status lina_popprof_save(const lina_pop_profile* prof, const char* path);
/* Shape of a profile (any output may be NULL). */
lina_status lina_popprof_info(const lina_pop_profile* prof, int32_t* num_layers, int32_t* num_experts,
                              int32_t* k, int32_t* path_len);
lina_status lina_popprof_load(const char* path, lina_pop_profile** out);
/* Phase two: *host_identical = 1 when the top-2k experts of the
 * estimate (host_estimated [E]) and of the actual selection counts
 * (host_actual_counts [E], e.g. the allgathered gate histogram) are the same set
 * (ranking by value desc, id asc; 2k capped at E), else 0 — then the caller re-plans
 * with lina_placement_compute on the actual popularity.  Errors: INVALID_ARGUMENT. */
lina_status lina_phase_two_check(const double* host_estimated, const int32_t* host_actual_counts,
                                 int32_t num_experts, int32_t k, int32_t* host_identical);

/* ------------------------------------------------------------------------ */
/* MoE layer                                                                 */
/* ------------------------------------------------------------------------ */
typedef struct {
  int32_t num_tokens;  /* T tokens on this rank (>= 0)                                  */
  int32_t d_model;     /* d  (d*elt % 16 == 0; bf16 also d % 128 == 0)                  */
  int32_t d_ffn;       /* f  (f*elt % 16 == 0; bf16 also f % 128 == 0)                  */
  int32_t num_experts; /* E global; static placement needs E % world == 0 (E_l = E/world) */
  int32_t k;           /* top-k, 1 <= k <= min(E, 8)  (k=2 training, k=1 inference) */
  int32_t capacity;    /* C >= 1 slots per expert per SOURCE rank (R5); C >= T => no drops, with
                          buffers padded to E·C rows per source.  0 = DROPLESS layout (§8(f) row 4):
                          no capacity bound; the per-expert counts are exchanged on the device and
                          the all-to-alls use an unequal split (P:525 applied to training), so the
                          receive buffers hold P·T·min(k, E_l) rows (plus one M tile per expert and
                          source) instead of E·T, and the source buffers T·k.  Needs n_chunks == 1;
                          across ranks: the fused transport, bf16, d and f multiples of 256, equal
                          num_tokens on every rank, world*E <= 512 (else UNSUPPORTED). */
  int32_t n_chunks;    /* all-to-all micro-ops per direction, 1 <= n <= C (R10) */
  lina_dtype dtype;    /* tokens, expert weights, outputs and their gradients            */
  int32_t pack;        /* expert packing factor m (0 or 1 = none): ranks form groups
                          of m consecutive ranks, every rank of group G hosts the same m·E/world
                          experts [G·m·E_l, (G+1)·m·E_l) (w1/w2/dw1/dw2 hold those m·E_l experts,
                          E_l = E/world), source rank s sends its rows of those experts to the
                          group member with rank % m == s % m (so a group's own rows stay on the
                          device), and the expert gradients are summed over the group (an NCCL
                          allreduce on a group communicator split off on first use).  m must
                          divide world; m > 1 runs on the variable layout (as capacity 0, with
                          or without a capacity bound) and has its requirements. */
} lina_moe_desc;

/* Optional routing tensors (device, caller-owned; NULL fields are skipped).
 * Forward writes them; with override_routing = 1, idx and gate are INPUTS
 * (caller-chosen routing: the paper's Ideal forced-balanced mode). */
typedef struct {
  int32_t* idx;     /* [T,k] selected experts, (logit desc, id asc) order (R3)   */
  float* gate;      /* [T,k] gate weights (R4)                                    */
  int32_t* slot;    /* [T,k] capacity slot, -1 = dropped (R5, R6)                 */
  int32_t* counts;  /* [E]   pre-drop assignments per expert from this rank       */
  float* probs;     /* [T,E] softmax probabilities                               */
  int32_t override_routing;
} lina_route;

/* Bytes of scratch (`workspace`) and of state kept from forward to backward
 * (`saved`) for this descriptor on this communicator.  saved may be 0-sized
 * pointer-wise for inference-only forward (pass saved = NULL).
 * Multi-rank rules (fused / copy-engine transports, where ranks store into and read
 * from each other's saved and workspace buffers):
 *   - capacity, n_chunks, num_experts, d_model, d_ffn and dtype must be equal on every
 *     rank; num_tokens may differ (every peer-visible region sits at an offset that does
 *     not depend on it).  The first call with a buffer checks this collectively and
 *     fails with INVALID_ARGUMENT on every rank otherwise.
 *   - saved and workspace are bound to the peers on their first use (a collective
 *     inside that call); a buffer freed and re-allocated is bound again, so all ranks
 *     must switch to new buffers in the same call (as an SPMD program does).
 *   - workspace is scratch: several layers on one communicator may share it (their
 *     calls are ordered by the per-communicator rounds); saved is per layer. */
lina_status lina_moe_workspace_size(const lina_comm* comm, const lina_moe_desc* desc,
                                    size_t* workspace_bytes, size_t* saved_bytes);

/* Training/inference forward with the static placement e -> rank floor(e/E_l):
 *   tokens [T,d] dtype; gate_w [d,E] fp32 (replicated); w1 [E_l,f,d], w2 [E_l,d,f]
 *   dtype (this rank's experts, nn.Linear layout); out [T,d] dtype = the MoE
 *   term only (the residual belongs to the caller, R7).  saved: NULL or
 *   saved_bytes (needed for backward).  n_chunks micro-ops per all-to-all,
 *   pipelined against the expert GEMMs.  Errors: INVALID_ARGUMENT,
 *   WORKSPACE, CUDA, NCCL. */
lina_status lina_moe_forward(lina_comm* comm, const lina_moe_desc* desc, const void* tokens,
                             const float* gate_w, const void* w1, const void* w2, void* out,
                             void* saved, void* workspace, size_t workspace_bytes,
                             lina_route* route, lina_stream stream);

/* Backward of lina_moe_forward (same desc, saved from that forward):
 *   dout [T,d] dtype -> dtokens [T,d] dtype; dgate_w [d,E] fp32 (this rank's
 *   sum over its tokens; the DP allreduce is lina_allreduce_submit's job, R12);
 *   dw1 [E_l,f,d], dw2 [E_l,d,f] dtype (sum over every source rank's tokens
 *   routed to this rank's experts).  No gradient flows through the top-k
 *   selection; dropped assignments get none (R13). */
lina_status lina_moe_backward(lina_comm* comm, const lina_moe_desc* desc, const void* saved,
                              const void* dout, const void* tokens, const float* gate_w,
                              const void* w1, const void* w2, void* dtokens, float* dgate_w,
                              void* dw1, void* dw2, void* workspace, size_t workspace_bytes,
                              lina_stream stream);

/* Inference forward with popularity-driven replication:
 *   w1_all [E,f,d], w2_all [E,d,f]: ALL experts on every rank (the paper keeps
 *   all experts in host DRAM; here in HBM so a placement change moves no
 *   weights).  placement: NULL => computed from this batch's global histogram
 *   (allreduce of per-expert counts; the paper's "w/o estimation" variant,
 *   P:905) with max_per_device; else used as given (e.g. an estimate-based
 *   plan, phase one).  plan_out (nullable, host arrays caller-allocated) gets the
 *   plan used.  Dropless top-k (capacity ignored, R5).  Synchronises the host
 *   once (H9).  Output equals lina_moe_forward's with a static placement (P9).
 *   A caller-supplied placement is checked entry by entry before use (its tables
 *   index device buffers): 1 <= replicas[e] <= min(world, max_replicas); replica
 *   devices in [0, world), distinct per expert, each hosting that expert; hosted ids
 *   in [-1, E), none twice on a device, each listed among its expert's replica
 *   devices.  INVALID_ARGUMENT lists every violation. */
lina_status lina_moe_infer_forward(lina_comm* comm, const lina_moe_desc* desc, const void* tokens,
                                   const float* gate_w, const void* w1_all, const void* w2_all,
                                   void* out, const lina_placement* placement,
                                   int32_t max_per_device, lina_placement* plan_out,
                                   void* workspace, size_t workspace_bytes, lina_stream stream);
/* Rows moved by the last lina_moe_infer_forward(_two_phase) call on this comm, as the
 * call's plan computed them (host copies; diagnostics and tests of the replica split,
 * R14): host_recv_rows[src] = rows this rank received from source rank src over all
 * its hosted experts; host_sent_rows[dv] = rows this rank sent to device dv.  Arrays
 * [world], host, caller-allocated, either may be NULL.  Before any inference call both
 * are zero.  Errors: INVALID_ARGUMENT for a NULL comm. */
lina_status lina_infer_last_rows(const lina_comm* comm, int32_t* host_recv_rows, int32_t* host_sent_rows);
/* Two-phase scheduling: as lina_moe_infer_forward with the phase-one
 * `placement` (built before gating from host_estimated [E], e.g. by
 * lina_popprof_estimate + lina_placement_compute), then, once the gate's global
 * per-expert counts are known, the phase-two check of lina_phase_two_check: the
 * top-2k experts of host_estimated and of the actual counts are compared as sets
 * and, if they differ, the plan is re-computed from the actual popularity ("following
 * the same logic in phase 1") before any token moves.  *host_replanned (may be
 * NULL) = 1 when phase two re-planned, else 0.  Every rank must pass the same
 * placement and host_estimated (e.g. the mean of the ranks' estimates, allgathered by
 * the caller); the decision and the final plan are then identical on every rank (the
 * counts are allgathered inside).  Errors: as lina_moe_infer_forward, plus
 * INVALID_ARGUMENT for a NULL placement or host_estimated, or a negative/NaN estimate. */
lina_status lina_moe_infer_forward_two_phase(lina_comm* comm, const lina_moe_desc* desc,
                                             const void* tokens, const float* gate_w,
                                             const void* w1_all, const void* w2_all, void* out,
                                             const lina_placement* placement,
                                             const double* host_estimated, lina_placement* plan_out,
                                             int32_t* host_replanned, void* workspace,
                                             size_t workspace_bytes, lina_stream stream);
/* Workspace for lina_moe_infer_forward with at most max_per_device hosted experts per
 * device (sized for the worst case: all of a source's tokens routed to one replica). */
lina_status lina_moe_infer_workspace_size(const lina_comm* comm, const lina_moe_desc* desc,
                                          int32_t max_per_device, size_t* workspace_bytes);

/* ------------------------------------------------------------------------ */
/* Micro-op allreduce scheduler (§4; §6.1)             */
/* ------------------------------------------------------------------------ */

/* policy and micro-op size (default LINA, 30 MB = the paper's partition). */
lina_status lina_sched_config(lina_comm* comm, lina_policy policy, size_t partition_bytes);
/* Queue one gradient (device, fp32 or bf16, `count` elements) for a SUM
 * allreduce over the DP communicator, in place.  It becomes ready when
 * `ready_stream` reaches this call.  Gradients are never mixed in one
 * micro-op.  Non-blocking. */
lina_status lina_allreduce_submit(lina_comm* comm, void* grad, size_t count, lina_dtype dtype,
                                  lina_stream ready_stream);
/* Make `stream` wait, on the device, until every allreduce submitted so far has
 * completed.  Does not block the host: the scheduler thread publishes the wait
 * point on its stream after the last micro-op (a stream memory write) and `stream`
 * waits for it (a stream memory wait), so the caller may enqueue further work at
 * once.  Not capturable in a CUDA graph (the micro-ops are issued later by the
 * scheduler thread).  An error of the scheduler thread surfaces here or at
 * lina_comm_check. */
lina_status lina_allreduce_wait(lina_comm* comm, lina_stream stream);
/* Scheduler statistics since the last call: micro-ops issued, micro-ops that
 * were deferred because an all-to-all was queued/in flight. */
lina_status lina_sched_stats(lina_comm* comm, int64_t* issued, int64_t* deferred);


/* ------------------------------------------------------------------------ */
/* Expert packing (§4.2; §6.1; §7.1; §8(f) row 3)          */
/* ------------------------------------------------------------------------ */
/* The packing rule: "starting with one expert per device, it iteratively increases the
 * number of experts per device in powers of two, until the FFN computation exceeds that
 * of the all-to-all micro-op": *pack_next = 2·pack when ffn_ms < a2a_ms and 2·pack
 * divides world, else pack.  Host only.  INVALID_ARGUMENT for pack not a power of two
 * dividing world, negative/NaN times or a NULL output. */
lina_status lina_pack_decide(int32_t world, int32_t pack, double ffn_ms, double a2a_ms, int32_t* pack_next);
/* The packing controller (host state): "adjusted after 10 training steps ...
 * every four steps".  Feed every training step's FFN and all-to-all micro-op times (e.g.
 * lina_profile gemm_ms / a2a_op_ms per step, the max over ranks so that every rank decides
 * the same); at step start_step and every `every` steps after, the means since the last
 * decision go through lina_pack_decide.  *pack = the factor to run with from the next step;
 * *changed (nullable) = 1 when it just changed (then re-pack the weights with
 * lina_pack_weights and run the layer with desc.pack = *pack). */
typedef struct lina_pack_ctl lina_pack_ctl;
lina_status lina_pack_ctl_create(int32_t world, int32_t start_step, int32_t every, lina_pack_ctl** out);
lina_status lina_pack_ctl_step(lina_pack_ctl* ctl, double ffn_ms, double a2a_ms, int32_t* pack, int32_t* changed);
lina_status lina_pack_ctl_destroy(lina_pack_ctl* ctl);
/* The one-time synchronous parameter exchange between packed devices: w_from
 * holds this rank's experts under pack_from ([m0·E_l][expert_elems], experts
 * [(rank/m0)·m0·E_l, ...)), w_to receives those under pack_to ([m1·E_l][expert_elems]);
 * each expert is copied from a rank hosting it under pack_from (itself when it can) over
 * peer memory.  Collective: every rank calls it with the same factors; the host blocks
 * (barrier before and after, so no rank changes w_from while another reads it).  Call
 * once per weight tensor (w1, w2).  Needs the fused or ce transport at world > 1. */
lina_status lina_pack_weights(lina_comm* comm, int32_t num_experts, int32_t pack_from, int32_t pack_to,
                              size_t expert_elems, lina_dtype dtype, const void* w_from, void* w_to,
                              lina_stream stream);

/* ------------------------------------------------------------------------ */
/* Instrumentation (bench.py / tests): counters since the last read.          */
/* ------------------------------------------------------------------------ */
typedef struct {
  int64_t kernel_launches; /* this library's CUDA kernel launches (all communicators, process-wide) */
  int64_t gemm_launches;   /* expert GEMM launches on this communicator while profiling   */
  double gemm_ms;          /* device time of the expert-GEMM phases (CUDA events recorded on the
                              compute stream around each phase, after its all-to-all waits) */
  int64_t gemm_phases;     /* number of timed phases summed into gemm_ms                  */
  double a2a_window_ms;    /* fused transport: summed all-to-all windows of the passes (first
                              mover launched on its stream .. last micro-op of the pass landed) */
  double gemm_in_a2a_ms;   /* expert-GEMM phase time inside those windows: / a2a_window_ms = the
                              paper's pipelining efficiency                            */
  int64_t a2a_windows;     /* number of windows summed                                      */
  double a2a_op_ms;        /* variable layout (capacity 0 / pack > 1): summed device time of the
                              all-to-all micro-ops themselves (count exchange + dispatch rows, and
                              the return rows, each up to the peers' READY) — the packing
                              controller's a2a micro-op time                         */
  int64_t a2a_ops;         /* number of micro-op intervals summed into a2a_op_ms             */
} lina_profile;

/* Bit flags: 1 = record timing events around the expert-GEMM phases of every forward /
 * backward on this communicator (cheap; off by default).  For the exposed-
 * communication measurement only (results are NOT valid while set, world > 1):
 * 2 = skip the all-to-all collectives (compute-only timing), 4 = run only the
 * all-to-all collectives of the pass (communication-only timing).  2 and 4 are
 * exclusive; 0 restores normal operation. */
lina_status lina_profile_enable(lina_comm* comm, int on);
/* Synchronises the recorded events, fills *out, and resets the counters. */
lina_status lina_profile_read(lina_comm* comm, lina_profile* out);

#ifdef __cplusplus
}
#endif
#endif /* LINA_H_ */
