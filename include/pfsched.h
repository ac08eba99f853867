/*
 * pfsched.h — C-ABI of libpfsched.so: the data-parallel hot path of the
 * Past-Future scheduler (Gong et al., arXiv 2507.10150), batched over many
 * independent scheduler instances, on NVIDIA B200 (sm_100a).
 *
 * Citations are PAPER.md line numbers of /root/reference/PAPER.md (LaTeX source)
 * with the LaTeX labels (Eq.(eq:5), Alg.(alg:sche), Eq.(eq:1)-(eq:3)); readings
 * of silent/ambiguous passages are numbered C-1..C-19 in DESIGN.md §3.
 *
 * The three calls of the paper's problem statement (Alg.1 inputs/outputs,
 * PAPER.md:212-213):
 *   pf_update_history  "records the actual output lengths of historical requests
 *                      ... L_h = {l_h^0..l_h^w} where w is the window size"
 *                      (Eq.(eq:5) PAPER.md:197-201)
 *   pf_estimate_peak   future required memory M* of the running batch,
 *                      Eq.(eq:1)-(eq:3), with each running
 *                      request's l̂ re-sampled from P(l > l_t) (Alg.1 lines 3-6,
 *                      PAPER.md:216-220)
 *   pf_admit           Alg.1 in full: predictions for running
 *                      and queued requests, then the longest FIFO queue prefix
 *                      whose M* fits the capacity M, early return at the first
 *                      failure
 *
 * Exact integer semantics (no floating point on the scheduling path; DESIGN.md §3 — only
 * the NEXT-3 analysis calls report fp64 cosines of exact integer Gram entries):
 *   history     w output lengths per window, FIFO; every value in [1, Lmax] (C-1, C-2)
 *   prediction  for a request with l_t generated tokens (l_t = 0 for queued, C-16):
 *               gt = sorted{h ∈ L_h : h > l_t} (C-4 strict); if gt is empty
 *               l̂ = max_new (C-5) else l̂ = gt[⌊u·|gt| / 2^32⌋] (C-3);
 *               l̂ = min(l̂, max_new) (C-6). With R repetitions the prediction
 *               is the max of the R samples (C-9).
 *   u           PF_MODE_QUANTILE: u = quantile_u for every request.
 *               PF_MODE_SAMPLE:   K = mix64(seed ^ tick·0xD1B54A32D192ED03 ^ inst·0x9E3779B97F4A7C15)
 *               u_rep = lowbias32(lo32(K) ^ hi32(K) ^ lo32((slot·R + rep)·0x9E3779B9)),
 *               u = max_rep u_rep; slot = s for the s-th running request (0-based),
 *               k + j − 1 for the j-th queued request (1-based); inst = global id (C-8).
 *   peak        a = l_p + l_t, r = l̂ − l_t; occupancy at tick τ ≥ 0 is
 *               O(τ) = Σ_{r_e ≥ τ} (a_e + τ) ("after growth, before removal",
 *               PAPER.md:262, C-10); M* = max_τ O(τ) = max_i (Σ_{j≤i} a_j + r_i·i)
 *               over the r-descending order (Eq.(eq:1)-(eq:3)); empty set → 0.
 *   admission   p* = the largest p ∈ [0, q] such that for every p' ≤ p
 *               10^4·M*(R ∪ Q[1..p']) ≤ (10^4 − reserved_bp)·M (C-12 '≤' PAPER.md:226,
 *               C-13 reserved ratio PAPER.md:342, C-14 early return PAPER.md:231).
 *               M* is monotone in p, so this is also the largest single p that fits.
 *
 * Conventions for every call:
 *   - Array arguments are caller-owned DEVICE pointers (e.g. torch tensor
 *     data_ptr()), int32 unless stated, densely packed. Inputs are read-only,
 *     outputs are fully overwritten; nothing is retained after the call.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream). All work is
 *     enqueued on it; no call synchronises the host except pf_create, pf_destroy,
 *     pf_get_device_error, pf_export_history, pf_sim_create, pf_sim_done,
 *     pf_sim_destroy and the two analysis calls (input check).
 *   - A context is not thread-safe; calls on one context must be stream-ordered.
 *   - Host-checkable problems return a negative pf_status synchronously and
 *     enqueue nothing; pf_last_error() then describes it (thread-local).
 *   - Data-dependent violations found on the device do not stop the call: the
 *     offending instance's outputs (or history row's update) are skipped/set to −1
 *     and a sticky device error word records the first (code, instance/row)
 *     (first writer wins) — read it with pf_get_device_error (PF_DERR_* codes).
 */
#ifndef PFSCHED_H
#define PFSCHED_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PF_ABI_VERSION 2

typedef struct pf_ctx pf_ctx;

typedef enum {
  PF_OK = 0,
  PF_EINVAL = -1,  /* NULL required pointer, bad size or parameter            */
  PF_ERANGE = -2,  /* declared bounds exceed what the kernels support/overflow */
  PF_ESTATE = -3,  /* call not valid in this context mode / sequence           */
  PF_ECUDA = -4,   /* a CUDA runtime call failed (message in pf_last_error)    */
  PF_ENCCL = -5,   /* NCCL missing or an NCCL call failed (shared mode)        */
  PF_ENOMEM = -6   /* device allocation failed                                 */
} pf_status;

enum { PF_MODE_SAMPLE = 0, PF_MODE_QUANTILE = 1 };
enum { PF_POLICY_AGGRESSIVE = 1, PF_POLICY_CONSERVATIVE = 2 };

/* Device error codes (sticky word, see pf_get_device_error). */
enum {
  PF_DERR_NONE = 0,
  PF_DERR_COMPLETION = 1,  /* completion length ∉ [1, Lmax]: that row is not updated    */
  PF_DERR_OFFSETS = 2,     /* CSR offsets decreasing or k+q > max_entries               */
  PF_DERR_MAX_NEW = 3,     /* max_new ∉ [1, Lmax]                                       */
  PF_DERR_INPUT_LEN = 4,   /* l_p ∉ [0, max_input_len]                                  */
  PF_DERR_GENERATED = 5,   /* l_t ∉ [0, max_new − 1]                                    */
  PF_DERR_CAPACITY = 6,    /* capacity < 0                                              */
  PF_DERR_OVERRIDE = 7     /* pf_admit_override: l̂ ∉ (l_t, Lmax] (running) or [1, Lmax] */
};

typedef struct {
  int32_t n_instances;     /* local instances on this device (>= 1)                            */
  int32_t window;          /* per-instance mode: w >= 1 per instance (C-1, default 1000,
                              PAPER.md:192/:295). Shared mode: the group's global window W,
                              W % 8 == 0, split into 8 shard rings of W/8 (C-18).               */
  int32_t max_len;         /* Lmax: output lengths live in [1, Lmax]; 1 <= Lmax <= 32767     */
  int32_t max_input_len;   /* declared bound on l_p (>= 0)                                    */
  int32_t max_entries;     /* declared bound on k+q per instance, 1..4096                     */
  int32_t n_groups;        /* 0 = per-instance histories; G > 0 = shared-group histories      */
  const int32_t* group_off;/* shared mode: device [G+1]; local instances of group g are
                              [group_off[g], group_off[g+1]) (group-major layout). Copied.     */
  int64_t instance_base;   /* per-instance mode: global id of local instance 0 (hash key)     */
  int32_t members_per_group; /* shared mode: global id of local instance l in group g is      */
  int32_t member_base;       /*   g·members_per_group + member_base + (l − group_off[g])      */
  int32_t mode;            /* PF_MODE_SAMPLE | PF_MODE_QUANTILE                               */
  uint32_t quantile_u;     /* u in quantile mode (0x80000000 = median rank)                   */
  int32_t repetitions;     /* R >= 1 (C-9); 0 = adaptive R = max(1, ⌈64/k⌉) per instance
                              (k = running batch size; SPEC.md:161 reading of PAPER.md:295) */
  int32_t reserved_bp;     /* reserved ratio in basis points, 0..9999 (C-13)                   */
  uint64_t seed;           /* sampling-mode seed (C-8)                                         */
  int32_t rank, nranks;    /* shared mode: this rank owns shards {s in 0..7 : s % nranks == rank} */
  const void* nccl_unique_id; /* shared mode, nullable: a 128-byte ncclUniqueId (from
                              pf_nccl_unique_id on one rank, the same bytes on every rank).
                              Set: the context owns an NCCL communicator of nranks ranks
                              (ncclCommInitRank in pf_create, collective) and
                              pf_update_history performs the all-reduce itself (also with
                              nranks == 1). NULL: with nranks > 1 the caller exchanges the
                              buffer (pf_exchange_buffer / pf_commit_history). Not retained. */
} pf_config;

/* Write a fresh ncclUniqueId (128 bytes) to id_out (host memory) for
 * pf_config.nccl_unique_id. Call on one rank and send the bytes to the others (any
 * out-of-band channel, e.g. a torch.distributed broadcast). NCCL is loaded at run time
 * (dlopen "libnccl.so.2", or $PFSCHED_NCCL_LIB); PF_ENCCL if it cannot be. */
pf_status pf_nccl_unique_id(void* id_out);

/* Create a context and its device history state.
 * init_history: device, oldest first, nullable (NULL ⇒ every slot = Lmax, C-2,
 *   "initialize the output length distribution using the preset maximum output
 *   length"). Layout: per-instance mode [n_instances × window];
 *   shared mode [G × shards_owned × W/8] in pf_update_history row order.
 *   Values must lie in [1, Lmax] (checked; PF_EINVAL otherwise).
 * Host-checked: n, w, Lmax, max_entries, R, reserved_bp, mode, rank/nranks
 *   ranges, nranks divides 8, and the int32 overflow bound
 *   max_entries·(max_input_len + 2·Lmax) < 2^31. The admit kernel's team of warps per
 *   instance keeps its tables in shared memory (per-instance histogram layout, w > Lmax+1:
 *   4·(Lmax+1) B of CDF + ≤ 10 B per request + bins); every size within these bounds fits
 *   one team (≤ 202 KB at Lmax = 32767, max_entries = 4096), and the one-warp variant packs
 *   fewer than 4 teams per CTA when 4 do not fit in 227 KB. Shared mode with nccl_unique_id: collective over the ranks (NCCL
 *   communicator creation + the first all-reduce); PF_ENCCL on NCCL failure.
 *   Synchronises `stream`. */
pf_status pf_create(const pf_config* cfg, const int32_t* init_history, void* stream,
                    pf_ctx** out);

/* Free all device state owned by the context (synchronises the device). */
pf_status pf_destroy(pf_ctx* ctx);

/* Record completed output lengths: for each history row, append
 * comp_len[comp_off[row] .. comp_off[row+1]) in order, evicting the oldest entry
 * whenever the row holds more than its window (FIFO, C-1). With more completions
 * than the window only the last `window` survive.
 * rows = n_instances (per-instance mode) or G·shards_owned (shared mode, rows
 * ordered group-major, owned shard minor). comp_off: device [rows+1], comp_len:
 * device [total]. A row containing a length ∉ [1, Lmax] is left unchanged and
 * PF_DERR_COMPLETION is recorded.
 * Shared mode: after the local update the owned-shard group histograms are
 * written to the exchange buffer. With a context-owned communicator
 * (nccl_unique_id) the call is COLLECTIVE: every rank calls it in the same order, and
 * it enqueues ncclAllReduce(sum, int32) of the buffer and the group-table rebuild on
 * `stream` (PF_ENCCL on NCCL failure). Without one: with nranks == 1 the group tables
 * are rebuilt here; with nranks > 1 the caller must sum-all-reduce the exchange buffer
 * across ranks (e.g. NCCL on `stream`) and then call pf_commit_history. */
pf_status pf_update_history(pf_ctx* ctx, const int32_t* comp_off, const int32_t* comp_len,
                            int32_t total, void* stream);

/* Shared mode only: the int32 [G × (Lmax+1)] device buffer that must be
 * all-reduced (sum) across ranks between pf_update_history and pf_commit_history.
 * Owned by the context. PF_ESTATE in per-instance mode. */
pf_status pf_exchange_buffer(pf_ctx* ctx, int32_t** buf, int64_t* count);

/* Shared mode only: rebuild the group CDF / sorted-window tables from the
 * (all-reduced) exchange buffer. No-op in per-instance mode; PF_ESTATE when the
 * context owns its communicator (pf_update_history already did it). Until the first
 * commit of a caller-exchanged context (nranks > 1, no nccl_unique_id),
 * pf_estimate_peak / pf_admit return PF_ESTATE.
 * The group tables are double-buffered: a rebuild (here, or inside
 * pf_update_history when nranks == 1) writes the half that the most recently
 * enqueued admit / estimate launch does NOT read, then makes it current for later
 * launches. So tick t+1's update / exchange / commit may run on a second stream
 * concurrently with tick t's admit, provided the rebuild for tick t+2 is ordered
 * after tick t's admit (the caller's events; bench.py does this). */
pf_status pf_commit_history(pf_ctx* ctx, void* stream);

/* M*(R) per instance (Eq.(eq:1)-(eq:3)) after re-predicting every running
 * request (Alg.1 lines 3-6). run_off: [n+1]; input_len, generated: [run_off[n]];
 * max_new: [n]; peak_out: [n]; pred_out: nullable [run_off[n]] = l̂ per running
 * request in input order. Equals pf_admit's peak_running_out for the same tick. */
pf_status pf_estimate_peak(pf_ctx* ctx, const int32_t* run_off, const int32_t* input_len,
                           const int32_t* generated, const int32_t* max_new, uint32_t tick,
                           int32_t* peak_out, int32_t* pred_out, void* stream);

/* Algorithm 1 per instance. q_off: [n+1], q_input_len: [q_off[n]] (FIFO order),
 * capacity: [n] (M, tokens). Outputs: admitted_out [n] = p*; peak_out [n] =
 * M*(R ∪ Q[1..p*]) (= M*(R) when p* = 0, which may exceed the capacity when the
 * running batch is already over-committed); peak_running_out nullable [n] = M*(R);
 * pred_run_out nullable [run_off[n]]; pred_q_out nullable [q_off[n]] (every queued
 * request, admitted or not). */
pf_status pf_admit(pf_ctx* ctx, const int32_t* run_off, const int32_t* input_len,
                   const int32_t* generated, const int32_t* q_off, const int32_t* q_input_len,
                   const int32_t* max_new, const int32_t* capacity, uint32_t tick,
                   int32_t* admitted_out, int32_t* peak_out, int32_t* peak_running_out,
                   int32_t* pred_run_out, int32_t* pred_q_out, void* stream);

/* Theoretical optimum (PAPER.md:341 "Theoretical optimum", :395: "the memory is
 * optimally utilized when the request output length is known"): Algorithm 1's
 * admission and Eq.(eq:1)-(eq:3) with the caller's l̂ per request instead of the
 * prediction (e.g. true output lengths). lhat_run: [run_off[n]], l_t < l̂ ≤ Lmax;
 * lhat_q: [q_off[n]], 1 ≤ l̂ ≤ Lmax; no max_new clamp. Outputs as pf_admit.
 * Violations give PF_DERR_OVERRIDE and −1 outputs for the instance. */
pf_status pf_admit_override(pf_ctx* ctx, const int32_t* run_off, const int32_t* input_len,
                            const int32_t* generated, const int32_t* lhat_run,
                            const int32_t* q_off, const int32_t* q_input_len,
                            const int32_t* lhat_q, const int32_t* capacity,
                            int32_t* admitted_out, int32_t* peak_out,
                            int32_t* peak_running_out, void* stream);

/* The paper's comparison policies (§5.3 Table 1),
 * batched on the same inputs, FIFO with early return:
 *   PF_POLICY_AGGRESSIVE   (watermark): admit the queue head while
 *       10^4·(Σ_running(l_p + l_t) + Σ_admitted l_p) ≤ ratio_bp·M
 *   PF_POLICY_CONSERVATIVE (overcommit, ":379 assumes 1.5 times"): admit while
 *       10^4·Σ_{running ∪ admitted}(l_p + max_new) ≤ ratio_bp·M
 * ratio_bp ≥ 1 (e.g. 9500 = watermark 95 %, 15000 = overcommit 150 %). Outputs:
 * admitted_out [n] = p*, used_out nullable [n] = the left-hand sum for the admitted set.
 * Validation and −1 outputs as pf_admit. Needs no history. */
pf_status pf_admit_baseline(pf_ctx* ctx, int32_t policy, int32_t ratio_bp, const int32_t* run_off,
                            const int32_t* input_len, const int32_t* generated,
                            const int32_t* q_off, const int32_t* q_input_len,
                            const int32_t* max_new, const int32_t* capacity,
                            int32_t* admitted_out, int32_t* used_out, void* stream);

/* Read (and keep) the sticky device error word; synchronises `stream`. */
pf_status pf_get_device_error(pf_ctx* ctx, int32_t* code, int32_t* index, void* stream);

/* Reset the sticky device error word (enqueued on `stream`). */
pf_status pf_clear_device_error(pf_ctx* ctx, void* stream);

/* Copy the history rings, oldest first, to device rows_out [rows × row_window]
 * (checkpoint / test hook; same layout as init_history). Enqueued on `stream`. */
pf_status pf_export_history(pf_ctx* ctx, int32_t* rows_out, void* stream);

/* ------------------------------------------------------------------------------------
 * Batched continuous-batching simulator: the serving loop the
 * paper's Table 1 measures ("Decoding Steps", "Current Consumed
 * Memory", "Future Required Memory", "Evicted Reqs"), one independent simulation per
 * instance, all instances advanced together on the device with the admission calls
 * above. Iteration semantics (readings S-1..S-9):
 *   S-1 every request of an instance is queued at t = 0 in list order;
 *   S-2 running requests with generated == true length finish; their lengths are
 *       recorded into the instance's window;
 *   S-3 admission over (running, the first min(|queue|, E − k) queued requests) by the
 *       policy: PF_SIM_PAST_FUTURE = pf_admit (tick = iteration index, reserved ratio
 *       param_bp); PF_SIM_OPTIMUM = pf_admit_override with the true lengths (the paper's
 *       "Theoretical optimum"; reserved param_bp); PF_SIM_AGGRESSIVE /
 *       PF_SIM_CONSERVATIVE = pf_admit_baseline (watermark / overcommit param_bp).
 *       A queued request enters with l_p + generated (evicted requests recompute);
 *   S-4 the admitted FIFO prefix joins the running list; an empty batch takes the queue
 *       head regardless (progress, counted as "forced");
 *   S-5 future-required sample: M* (Eq.(eq:1)-(eq:3)) of the running set with TRUE
 *       remaining lengths;
 *   S-6 while Σ(l_p + l_t) + k > M and k > 1: evict the most recently admitted request,
 *       re-queue it at the FRONT with its generated tokens (LIFO);
 *   S-7 decode: every running request gains one token;
 *   S-8 consumed sample Σ(l_p + l_t);  S-9 done when queue and batch are empty.
 * Metrics per instance (int64, PF_SIM_NMETRICS columns): iterations, decoding steps,
 * evictions, finished requests, Σ consumed, Σ future, samples, max future, forced
 * admissions, admissions. Averages / capacity give Table 1's percentages. */
typedef struct pf_sim pf_sim;
enum { PF_SIM_PAST_FUTURE = 0, PF_SIM_OPTIMUM = 1, PF_SIM_AGGRESSIVE = 2,
       PF_SIM_CONSERVATIVE = 3 };
#define PF_SIM_NMETRICS 10

typedef struct {
  int32_t n_instances;    /* independent simulations (>= 1)                              */
  int32_t window;         /* history window w of each instance (C-1)                      */
  int32_t max_len;        /* Lmax >= every max_new (C-2 initial window value)             */
  int32_t max_input_len;  /* bound on request input lengths                              */
  int32_t max_entries;    /* E: running + admission window per instance, 1..4096          */
  int32_t policy;         /* PF_SIM_*                                                     */
  int32_t param_bp;       /* reserved bp (0..9999) | watermark / overcommit bp (>= 1)     */
  int32_t mode;           /* past-future prediction: PF_MODE_SAMPLE | PF_MODE_QUANTILE    */
  uint32_t quantile_u;
  int32_t repetitions;    /* R (C-9), 0 = adaptive                                        */
  uint64_t seed;
  int64_t instance_base;  /* hash key of instance i = instance_base + i (C-8)              */
} pf_sim_config;

/* Create a simulator. Device arrays (copied; the caller keeps ownership):
 *   req_off [n+1] (requests of instance i are [req_off[i], req_off[i+1]), list order),
 *   req_input / req_output [req_off[n]] (l_p in [0, max_input_len], true output length
 *   in [1, max_new[i]]), max_new [n] in [1, max_len], capacity [n] (M, tokens, with
 *   l_p + L <= M for every request), init_history [n × window] nullable (oldest first;
 *   NULL ⇒ Lmax, C-2). Host-validated (synchronises `stream`); PF_EINVAL on violation. */
pf_status pf_sim_create(const pf_sim_config* cfg, const int32_t* req_off,
                        const int32_t* req_input, const int32_t* req_output,
                        const int32_t* max_new, const int32_t* capacity,
                        const int32_t* init_history, void* stream, pf_sim** out);

/* Advance every instance by `iterations` iterations (finished instances idle). Enqueued.
 * With iterations >= 4 the iterations are replayed from CUDA graphs of 1 and 8
 * iterations, captured on the first such call on a private stream (the admission tick
 * of each replay is set on the graph's admit nodes); the results are identical to
 * plain launches. The graphs live until pf_sim_destroy. */
pf_status pf_sim_step(pf_sim* sim, int32_t iterations, void* stream);

/* Number of finished instances (synchronises `stream`). */
pf_status pf_sim_done(pf_sim* sim, int32_t* n_done, void* stream);

/* Copy metrics [n × PF_SIM_NMETRICS] int64 and, if non-NULL, generated tokens and
 * eviction counts per request [req_off[n]] to device buffers. Enqueued. */
pf_status pf_sim_metrics(pf_sim* sim, int64_t* metrics_out, int32_t* generated_out,
                         int32_t* evictions_out, void* stream);

/* The simulator's library context (device error word, history export). */
pf_ctx* pf_sim_context(pf_sim* sim);

pf_status pf_sim_destroy(pf_sim* sim);

/* ------------------------------------------------------------------------------------
 * Window-similarity analysis (fig:dist / fig:cos_win,
 * PAPER.md:175-192): how similar the output-length distributions of request windows are.
 * `lengths` is a device stream of output lengths in [1, max_len] (checked: PF_EINVAL;
 * these calls synchronise `stream` for the check). Windows are consecutive,
 * non-overlapping blocks of `window` requests, the trailing remainder dropped
 * (fig:dist caption "1000 requests, no overlap"); h_b(l) counts length l in window b
 * (token-exact bins).
 *   pf_window_similarity: B = n / window >= 2 windows.
 *     gram_out    [B × B] int64 (nullable): G[i][j] = Σ_l h_i(l)·h_j(l), exact
 *     cos_out     [B × B] fp64  (nullable): G[i][j] / sqrt(G[i][i]·G[j][j])
 *     summary_out [2]     fp64  (nullable): mean_i cos[i][i+1] ("diagonal"),
 *                                           mean_{i≠j} cos[i][j] ("global")
 *   pf_adjacent_similarity: a historical window of hist_window requests followed by a
 *     running window of run_window: running window k = [h + k·r, h + (k+1)·r),
 *     K = (n − h) / r; cos_out [K] fp64 = cosine of (historical_k, running_k);
 *     mean_out [1] fp64 nullable = their mean. */
pf_status pf_window_similarity(const int32_t* lengths, int64_t n, int32_t window, int32_t max_len,
                               int64_t* gram_out, double* cos_out, double* summary_out,
                               void* stream);
pf_status pf_adjacent_similarity(const int32_t* lengths, int64_t n, int32_t hist_window,
                                 int32_t run_window, int32_t max_len, double* cos_out,
                                 double* mean_out, void* stream);

/* ------------------------------------------------------------------------------------
 * Cross-instance request forwarding by M* headroom (the paper's
 * future work: "forward requests to underutilized services ... aiming to
 * ensure that each service reaches full capacity"). Readings F-1..F-4:
 * the context's n_instances are n / cluster_size clusters of cluster_size instances
 * (instance s of cluster c = c·cluster_size + s), each cluster with one FIFO queue
 * (cq_off [C+1], cq_input_len). Requests are forwarded in queue order; request j goes
 * to the instance s that passes Alg.1's check 10^4·M*_s(R_s ∪ F_s ∪ {j}) ≤
 * (10^4 − reserved_bp)·M_s with the largest headroom (ties: lowest s); the first
 * request no instance can take stops forwarding (C-14). Predictions per instance are
 * pf_admit's: running slots 0..k_s−1, the cluster's j-th queued request (1-based) as
 * slot k_s + j − 1 (C-8, R = 1). Outputs: dest_out [cq_off[C]] = instance in [0, S) or
 * −1; forwarded_out [C]; peak_out [n] = M*_s(R_s ∪ F_s). Needs a per-instance context
 * with window <= Lmax + 1 (PF_ESTATE otherwise), cluster_size in [1, 32] dividing n,
 * cluster_size·max_entries·8 <= 200 KB (PF_ERANGE). Data errors: the cluster's outputs
 * are −1 and the sticky device error word is set. Enqueued on `stream`. */
pf_status pf_forward(pf_ctx* ctx, int32_t cluster_size, const int32_t* run_off,
                     const int32_t* input_len, const int32_t* generated, const int32_t* max_new,
                     const int32_t* capacity, const int32_t* cq_off, const int32_t* cq_input_len,
                     uint32_t tick, int32_t* dest_out, int32_t* forwarded_out, int32_t* peak_out,
                     void* stream);

/* Describes the last failing call on this thread ("" if none). */
const char* pf_last_error(void);

int32_t pf_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PFSCHED_H */
