/* asc.h — C ABI of the B200-native Ascendra scheduler / batch-level simulator hot path.
 *
 * Method: Ascendra, "Dynamic Request Prioritization for Efficient LLM Serving"
 * (arXiv 2504.20828).  Citations: P:n = PAPER.md line n (LaTeX source), S:n = SPEC.md line n,
 * Gnn = reading nn in DESIGN.md §Readings (where the paper is silent or garbled).
 *
 * Library: paper_2504_20828_b200/libasc.so (sm_100a CUDA kernels; no CPU fallback).
 *
 * Conventions for every entry point
 *  - Time is int64 microseconds; token counts are int32; F (flops) and M (bytes) are exact
 *    integers < 2^53 evaluated inside the kernels (G18).
 *  - Array arguments are plain pointers.  asc_schedule_step, asc_simulate_batch and asc_goodput
 *    accept DEVICE pointers (memory on the ctx's device, e.g. torch tensors' data_ptr()) or HOST
 *    pointers (pageable or pinned); host arrays are staged through the ctx's device workspace
 *    inside the call (uploads before, downloads after).  All arrays of one call must be of the
 *    same kind (all host or all device), else ASC_E_INVAL.
 *  - The caller owns every input and output array.  The ctx owns its device workspace, grows it
 *    on demand (ASC_E_NOMEM if that fails) and frees it in asc_destroy.
 *  - Calls enqueue on the stream bound at asc_create and synchronize before returning, so the
 *    status reflects kernel errors and device-side invariant checks.  One ctx per host thread.
 *  - No partial results are guaranteed on error.  asc_last_error(ctx) names the offending field
 *    or check (asc_last_error(NULL) reports asc_create failures of the calling thread).
 */
#ifndef ASC_H
#define ASC_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define ASC_ABI_VERSION 3
#define ASC_MAX_BATCH 128      /* max request-count budget R / lp_max_batch */
#define ASC_MAX_INSTANCES 16   /* n_lp + n_hp per trace */

typedef struct asc_ctx asc_ctx;

typedef enum {
  ASC_OK = 0,
  ASC_E_INVAL = 1,      /* bad argument (NULL, negative size, unsorted arrivals, mixed pointers) */
  ASC_E_CONFIG = 2,     /* configuration / liveness validation failed (field named) */
  ASC_E_NOMEM = 3,      /* device workspace allocation failed */
  ASC_E_CUDA = 4,       /* CUDA runtime error (message from cudaGetErrorString) */
  ASC_E_EMPTY = 5,      /* goodput over a trace with 0 requests */
  ASC_E_RANGE = 6,      /* F or M >= 2^53, R > ASC_MAX_BATCH, index >= 2^31 */
  ASC_E_INVARIANT = 7   /* device-side invariant violated (KV ledger, stuck queue) */
} asc_status;

/* Value function pi (G19).  key ascending = priority descending; ties by ascending id.
 *  EDF_LAXITY   key = deadline - prefill_us   (default: urgency grows with time in system and
 *                                              prompt length)
 *  EDF_DEADLINE key = deadline = arrival + TTFT SLO
 *  SJF          key = prefill_us
 *  LJF          key = -prefill_us
 *  FCFS         key = arrival  (asc_schedule_step: entry position)
 *  WEIGHTED     key = key_w[0]*deadline + key_w[1]*prefill_us + key_w[2]*arrival: an operator
 *               value function ("any customized policy"; row f4, G51);
 *               asc_simulate_batch only.
 * asc_simulate_batch adds asc_traces.req_key_offset_us[i] (when given) to request i's key under
 * every policy: service classes, e.g. premium users ahead of the free tier. */
typedef enum {
  ASC_POLICY_EDF_LAXITY = 0, ASC_POLICY_EDF_DEADLINE = 1, ASC_POLICY_SJF = 2,
  ASC_POLICY_LJF = 3, ASC_POLICY_FCFS = 4, ASC_POLICY_WEIGHTED = 5
} asc_policy;

/* Model symbols (App. A.1): hidden h, heads n, head size s (h = n*s), KV heads n_kv,
 * FFN size m, layers L (G11), attention block size b (G15), bytes per element (G10), tensor
 * parallel degree tp (h, n, m, n_kv are divided by tp). */
typedef struct { int32_t h, n, s, n_kv, m, L, b, dtype_bytes, tp; } asc_arch;

/* Latency regression (Eq. 4-5): t = C1(tM+tF) + C2 max(tM,tF) + C3 tM + C4 tF + C5,
 * tM = M/M_H, tF = F/F_H (seconds; M_H bytes/s, F_H flops/s). */
typedef struct { double c[5]; double F_H, M_H; } asc_perf;

/* Instance partition and budgets (G22, G32, G38). */
typedef struct {
  int32_t n_lp, n_hp;            /* LP (throughput) and HP (latency) instances per trace */
  int32_t block_tokens;          /* KV block size in tokens (G32) */
  int32_t kv_blocks_lp, kv_blocks_hp; /* KV capacity per instance in blocks */
  int32_t lp_max_batch;          /* LP batch cap, <= ASC_MAX_BATCH */
  int32_t lp_token_budget;       /* N of Algorithm 1 (G38) */
  int32_t hp_token_budget;       /* HP base prefill token budget; also sizes W_hp */
} asc_topology;

/* Switches (P:336 offload, P:368 tickets, P:370-371 elastic, P:373-375 drop). */
typedef struct {
  int32_t policy;                /* asc_policy */
  uint8_t offload, tickets, elastic, drop;
  int64_t offload_margin_us;     /* tunable threshold of P:336 (G24), default 0 */
  int64_t offload_delay_us;      /* LP->HP transfer delay, default 0 */
  int32_t hist_default_tokens;   /* decode-length history mean before any HP completion (G28) */
  int32_t scheduler;             /* asc_scheduler: Ascendra, or a baseline on n_lp homogeneous
                                    instances (requires n_hp = 0, DESIGN G46-G48) */
  int32_t chunk_tokens;          /* ASC_SCHED_SARATHI: per-batch token budget, decodes + prefill
                                    chunks (G47; in [1, 2^24)); ignored otherwise */
  int32_t offload_rule;          /* 0: the paper's rule: deadline - T <= prefill_us + W_hp
                                    + margin.  1: look-ahead (row f4, G50): + the prefill_us of
                                    every waiting request ahead in priority order.
                                    asc_simulate_batch only (asc_schedule_step: ASC_E_CONFIG) */
  int32_t key_w[3];              /* ASC_POLICY_WEIGHTED weights, each in [-1024, 1024] */
} asc_flags;

/* Schedulers asc_simulate_batch can run.  ASC_SCHED_VLLM is the vLLM-like baseline the paper
 * compares against ("prefill-prioritizing"): every instance orders its
 * waiting queue by the policy key (FCFS = vLLM), runs a prefill-only batch of the longest prefix
 * fitting lp_token_budget (<=), the free KV blocks and lp_max_batch whenever one fits (ongoing
 * decodes stall), else one decode-only step of every running request (preemption by
 * recomputation).  ASC_SCHED_SARATHI is the Sarathi-like chunked-prefill baseline (
 * S:392-400; App. A.4 cost): every decode runs each batch and the rest of
 * chunk_tokens is filled with prefill chunks in queue order (a partially prefilled request is
 * continued first), each request taking min(budget left, prompt left).  asc_schedule_step is
 * Ascendra's LP decision and ignores this field. */
typedef enum { ASC_SCHED_ASCENDRA = 0, ASC_SCHED_VLLM = 1, ASC_SCHED_SARATHI = 2 } asc_scheduler;

typedef struct { asc_arch arch; asc_perf perf; asc_topology topo; asc_flags flags; } asc_config;

/* Validates cfg (ASC_E_CONFIG naming the field: h != n*s, tp divisibility, non-positive sizes,
 * F_H/M_H <= 0, lp_max_batch > ASC_MAX_BATCH, n_lp < 1, n_lp + n_hp > ASC_MAX_INSTANCES),
 * binds device `device` and stream `cuda_stream` (a cudaStream_t; NULL = legacy default
 * stream), and precomputes the per-prompt-length prefill latency table on the device. */
asc_status asc_create(const asc_config* cfg, int device, void* cuda_stream, asc_ctx** out);
void asc_destroy(asc_ctx* ctx);
const char* asc_last_error(const asc_ctx* ctx);
int32_t asc_abi_version(void);

/* ---------------------------------------------------------------------------------------------
 * asc_schedule_step — one stateless LP scheduling decision for each of S independent segments
 * (a segment = the waiting queue of one LP instance of one trace), i.e. §5 of the paper for one
 * batch-formation instant: per request the performance model (Eq. 1-5) gives prefill_us and the
 * KV blocks blk = ceil((p+1)/block_tokens) (G23); the value function gives the key; Algorithm 1
 * admits the longest prefix of the key order whose running token, block and
 * microsecond sums stay strictly below N, M and C with at most R requests (G21-G22); the offload
 * rule (G24) flags the remaining never-prefilled, not-on-HP requests with
 * deadline - now <= prefill_us + W_hp + margin (W_hp = prefill latency of hp_token_budget tokens);
 * with the drop flag, never-prefilled requests with now > deadline are dropped first (G34)
 * and take no further part.  C = tbt_slo - latency(decode-only batch of dec_count requests with
 * context sum dec_ctx_sum), or +infinity when dec_count = 0 (G22).  batch_lat_us = latency of
 * the hybrid batch {admitted prefills} + {decodes} (Eq. 3-5), 0 when both are empty.
 *
 * Layout: entries of segment s are [seg_off[s], seg_off[s+1]) of the per-entry arrays, in
 * ascending request-id (arrival) order; ties in the key order break by position.  Outputs use the
 * same CSR offsets: admit_idx[seg_off[s] + j], j < admit_cnt[s] (priority order); offload_idx and
 * drop_idx likewise (ascending position).  Indices are global entry positions (int32).
 * flags: bit0 = ever prefilled (preempted request), bit1 = already on an HP.
 * Errors: ASC_E_INVAL (S < 0, seg_off not non-decreasing, eff_prompt < 1, dec_count > 0 with
 * dec_ctx_sum < dec_count), ASC_E_RANGE
 * (budget_reqs > ASC_MAX_BATCH, total entries >= 2^31, eff_prompt >= 2^24, a cost F or M >= 2^53
 * -- detected even where the uint64 products would wrap, e.g. a huge dec_ctx_sum).
 * ------------------------------------------------------------------------------------------- */
typedef struct {
  int32_t S;
  int64_t Q;                     /* total entries = seg_off[S]; -1: the library reads it (one
                                    device->host copy of 8 bytes for device arrays) */
  const int64_t* seg_off;        /* [S+1] */
  const int64_t* now_us;         /* [S] */
  const int64_t* deadline_us;    /* [Q] arrival + TTFT SLO */
  const int32_t* eff_prompt;     /* [Q] prompt (+ generated tokens after preemption), >= 1 */
  const uint8_t* flags;          /* [Q] */
  const int32_t* dec_count;      /* [S] B_d */
  const int64_t* dec_ctx_sum;    /* [S] sum of decode contexts lhat, >= dec_count; ignored when dec_count = 0 */
  const int64_t* tbt_slo_us;     /* [S] */
  const int32_t* budget_tokens;  /* [S] N */
  const int32_t* budget_blocks;  /* [S] M (free KV blocks) */
  const int32_t* budget_reqs;    /* [S] R (<= ASC_MAX_BATCH) */
} asc_step_in;

typedef struct {
  int32_t* admit_idx;   int32_t* admit_cnt;     /* [Q] CSR, [S] */
  int32_t* offload_idx; int32_t* offload_cnt;   /* [Q] CSR, [S] */
  int32_t* drop_idx;    int32_t* drop_cnt;      /* [Q] CSR, [S] */
  int64_t* batch_lat_us;                        /* [S] */
  int32_t* prefill_us;                          /* [Q] optional (NULL = not written) */
} asc_step_out;

asc_status asc_schedule_step(asc_ctx* ctx, const asc_step_in* in, asc_step_out* out);

/* ---------------------------------------------------------------------------------------------
 * asc_simulate_batch — batch-level discrete-event simulation (§4-§6; the paper's simulator of
 * P:377/P:630) of T independent traces, each on its own n_lp + n_hp instances, with the event
 * rules of DESIGN.md §Event loop: completions, offload deliveries, arrivals (round-robin to LPs or
 * to a ticket-holding HP), formations (LP: drop, decode growth with LIFO preemption by
 * recomputation, Algorithm 1, offload, hybrid batch; HP: drop, FCFS prefill-first under the
 * (elastic) token limit, else decode-only), then ticket issue.
 *
 * Layout: requests of trace t are [trace_off[t], trace_off[t+1]) in arrival order (arrival_us
 * non-decreasing within a trace, else ASC_E_INVAL).  Per-trace SLOs; req_ttft_slo_us optionally
 * overrides the TTFT SLO per request (NULL = per-trace).  Liveness validation (ASC_E_CONFIG):
 * prompt_len, output_len >= 1; prompt_len + output_len <= lp_token_budget; and
 * ceil((prompt_len + output_len)/block_tokens) < min KV blocks of the instances.
 * Outputs per request: first_token_us (TTFT event), done_us (completion), prefill_start_us
 * (first admission), -1 when absent; status bits 0-1 state {0 unfinished, 1 completed,
 * 2 dropped}, bit 2 offloaded, bit 3 ticketed, bits 4-11 serving instance (255 = none),
 * bits 12-27 preemptions.  Per trace: digest, decisions (non-empty
 * formations) and evaluations (waiting-queue entries examined, summed over formations);
 * decisions/evaluations may be NULL.
 * ------------------------------------------------------------------------------------------- */
typedef struct {
  int32_t T;
  int64_t R;                       /* total requests = trace_off[T]; -1: the library reads it */
  const int64_t* trace_off;        /* [T+1] */
  const int64_t* arrival_us;       /* [R] */
  const int32_t* prompt_len;       /* [R] */
  const int32_t* output_len;       /* [R] */
  const int64_t* ttft_slo_us;      /* [T] (Table 2) */
  const int64_t* tbt_slo_us;       /* [T] */
  const int64_t* req_ttft_slo_us;  /* [R] optional */
  const int32_t* n_lp;             /* [T] optional per-trace subgroup topology (row
                                      f3): trace t runs on n_lp[t] LP + n_hp[t] HP instances; */
  const int32_t* n_hp;             /* n_lp >= 1, n_hp >= 0, n_lp + n_hp <= the ctx's n_lp + n_hp
                                      (ASC_E_CONFIG otherwise); NULL = the ctx's topology */
  const int64_t* req_key_offset_us; /* [R] optional value-function offset per request (service
                                      class, G51): added to the policy key; |offset| < 2^40 */
} asc_traces;

typedef struct {
  int64_t* first_token_us;  /* [R] */
  int64_t* done_us;         /* [R] */
  int64_t* prefill_start_us;/* [R] */
  uint32_t* status;         /* [R] */
  uint64_t* digest;         /* [T] */
  int64_t* decisions;       /* [T] optional */
  int64_t* evaluations;     /* [T] optional */
} asc_outcomes;

asc_status asc_simulate_batch(asc_ctx* ctx, const asc_traces* tr, asc_outcomes* out);

/* Diagnostics: decision snapshots of the simulator (SURVEY §8(d) config-4 self-check: "sampled
 * formations replayed through asc_schedule_step must equal the simulator's admissions").  Arms the
 * NEXT asc_simulate_batch on ctx (device-pointer calls only) to record, at every Algorithm-1 LP
 * formation of LP instance `instance` of trace `trace` whose ordinal o (1 + the formations of that
 * instance recorded in its digest so far) is a multiple of `every`, the inputs the decision used
 * and the decision it made:
 *   hdr[16 s + 0..14] = T (now), instance, N (lp_token_budget), M (free KV blocks after decode
 *     preparation), B_d (decodes), sum of their contexts, tbt SLO, R (lp_max_batch - B_d), queue
 *     length q, first entry in the entry arrays, admitted count, offloaded count, first id in
 *     out_ids, batch latency (µs), o;
 *   ids / deadline_us / eff_prompt / flags [e0, e0 + q): the waiting queue in the simulator's
 *     (key, id) order: request id within the trace, deadline, effective prompt, bit0 = ever
 *     prefilled, bit1 = on an HP -- exactly asc_schedule_step's per-entry inputs;
 *   out_ids [o0, o0 + admitted + offloaded): admitted ids in priority order, then offloaded ids
 *     ascending.
 * Snapshots stop when max_snaps, entry_cap or out_cap would be exceeded; counts[0..2] (device,
 * int64) receive the snapshots, entries and out ids used.  The arming is consumed by the next
 * asc_simulate_batch.  All pointers are device memory owned by the caller. */
typedef struct {
  int32_t trace, instance;
  int64_t every;
  int32_t max_snaps;
  int64_t entry_cap, out_cap;
  int64_t *hdr, *counts;
  int32_t* ids;
  int64_t* deadline_us;
  int32_t* eff_prompt;
  uint8_t* flags;
  int32_t* out_ids;
} asc_snapshots;
asc_status asc_arm_snapshots(asc_ctx* ctx, const asc_snapshots* snap);

/* ---------------------------------------------------------------------------------------------
 * asc_goodput — per trace, good = #requests that COMPLETED with first_token - arrival <= TTFT SLO
 * and (output_len = 1 or done - first_token <= TBT SLO * (output_len - 1)), i.e. mean TBT within
 * the SLO (G35); total = all requests including dropped/unfinished (G36).
 * Exact integers so sums across GPUs are exact.  ASC_E_EMPTY if some trace has 0 requests.
 * ------------------------------------------------------------------------------------------- */
asc_status asc_goodput(asc_ctx* ctx, const asc_traces* tr, const asc_outcomes* out,
                       uint64_t* good, uint64_t* total);

/* ---------------------------------------------------------------------------------------------
 * asc_summarize — the per-trace outcome summary behind the paper's metrics (row a8): PAPER
 * P:579-584 (Fig. 10: "(a) P99 TTFT, (b) Mean TBT, (c) System throughput, and (d) Request
 * scheduling delay"; "HP requests wait 4x less than LP requests"), SPEC S:543-590 (metrics
 * module), reading G52.  For each trace t (every output is an int64 [T] array and may
 * be NULL = not written):
 *   completed, dropped   requests whose status state is COMPLETED / DROPPED
 *   violating            completed requests that are not good (asc_goodput's test failed)
 *   tokens               sum of output_len over completed requests (dropped contribute 0);
 *                        system throughput = tokens / (last_done_us - first arrival)
 *   ttft_p50_us, ttft_p90_us, ttft_p99_us
 *                        nearest-rank percentiles (the ceil(q n / 100)-th smallest) of
 *                        first_token_us - arrival_us over the n requests with a first token;
 *                        -1 when n = 0
 *   tbt_sum_us, tbt_tokens
 *                        sums of done - first_token and of output_len - 1 over completed
 *                        requests with output_len > 1: mean TBT = tbt_sum_us / tbt_tokens
 *   delay_sum_lp_us, delay_cnt_lp, delay_sum_hp_us, delay_cnt_hp
 *                        scheduling delay prefill_start_us - arrival_us summed and counted over
 *                        requests with a prefill start, split by the type of the serving
 *                        instance in the status word (index < n_lp of the trace: LP, else HP)
 *   last_done_us         the latest done_us among completed requests (-1 if none)
 * Inputs: tr (trace_off, arrival_us, output_len, ttft_slo_us, tbt_slo_us, optional
 * req_ttft_slo_us and per-trace n_lp) and out (first_token_us, done_us, prefill_start_us,
 * status) as produced by asc_simulate_batch.  All pointers device, or all host (staged).
 * Exact integers, so per-trace results equal the CPU oracle's and sums over GPUs are exact.
 * Errors: ASC_E_INVAL (NULL inputs, T < 0, mixed pointer kinds).
 * ------------------------------------------------------------------------------------------- */
typedef struct {
  int64_t *completed, *dropped, *violating, *tokens;
  int64_t *ttft_p50_us, *ttft_p90_us, *ttft_p99_us;
  int64_t *tbt_sum_us, *tbt_tokens;
  int64_t *delay_sum_lp_us, *delay_cnt_lp, *delay_sum_hp_us, *delay_cnt_hp;
  int64_t *last_done_us;
} asc_summary;
asc_status asc_summarize(asc_ctx* ctx, const asc_traces* tr, const asc_outcomes* out,
                         asc_summary* sum);

/* Diagnostics: number of libasc kernels the last call on ctx launched (bench evidence). */
int64_t asc_last_kernel_launches(const asc_ctx* ctx);
/* Diagnostics: device time (ms, CUDA events on the ctx stream) of the last call's dominant
 * kernel (simulate: the step loop; schedule_step: the streaming pass; goodput: the reduction),
 * or -1 if none ran. */
double asc_last_kernel_ms(const asc_ctx* ctx);
/* Diagnostics: device time (ms) of the last call's secondary kernel (schedule_step: k_lane, the
 * one-thread-per-segment pass over segments of <= 32 entries), or -1 if the call has none. */
double asc_last_kernel2_ms(const asc_ctx* ctx);

/* ---------------------------------------------------------------------------------------------
 * asc_fit_perf — batched calibration of the performance model.
 * PAPER P:273-277 (Eq. 4-5: "perform a linear regression to find the corresponding parameters
 * C1 ... C5") and P:279 (runtime logs of each batch periodically refit the model); solver and
 * regularisation are readings (DESIGN G49).  For each of G independent groups of
 * batch records (CSR rec_off, group g = records [rec_off[g], rec_off[g+1])): record i has the
 * batch's exact flop count F[i] and byte count M[i] (as the cost model gives them) and its
 * observed latency y[i] in seconds (> 0).  With tM = M / M_H, tF = F / F_H (the ctx's perf caps)
 * and x = (tM + tF, max(tM, tF), tM, tF, 1), returns the ridge least-squares coefficients
 *     coef[5g .. 5g+4] = argmin_c  sum_i (x_i . c - y_i)^2 + lambda |c|^2      (C1 .. C5)
 * solved from the normal equations by Cholesky (lambda > 0 breaks the exact x1 = x3 + x4
 * collinearity; compare predictions, not coefficients).  mean_err / max_err (each may be NULL):
 * in-sample mean and max of |pred - y| / y, pred = the fitted Eq. 4-5 clamped at 0.
 * Layout: SoA arrays, all device pointers or all host pointers (host arrays are staged).
 * Errors: ASC_E_INVAL (NULL arrays, lambda < 0 or not finite, y <= 0), ASC_E_EMPTY (a group with
 * fewer than 20 records), ASC_E_RANGE (system not positive definite).  Results are
 * deterministic (fixed reduction order); they match a sequential CPU sum to rounding. */
typedef struct {
  int32_t G;                 /* independent fits */
  int64_t N;                 /* total records = rec_off[G]; -1 = read it from rec_off */
  const int64_t* rec_off;    /* [G+1] non-decreasing, rec_off[0] = 0 */
  const uint64_t* F;         /* [N] flops of the batch */
  const uint64_t* M;         /* [N] bytes of the batch */
  const double* y;           /* [N] observed seconds */
} asc_fit_in;
asc_status asc_fit_perf(asc_ctx* ctx, const asc_fit_in* in, double lambda, double* coef,
                        double* mean_err, double* max_err);

/* ---------------------------------------------------------------------------------------------
 * asc_latency — the performance model's latency of n batches given their exact costs (rows
 * a1/a6, the evaluation every formation makes).  PAPER P:273-277 (Eq. 4-5: t = C1(tM + tF) +
 * C2 max(tM, tF) + C3 tM + C4 tF + C5 with tM = M / M_H, tF = F / F_H), readings G17 (clamp at 0,
 * S:187; at least 1 µs) and G18 (ceil to integer microseconds).  For i < n:
 *     t_s[i]    = max(0, t(F[i], M[i]))      seconds, every fp64 op round-to-nearest in the order
 *                                            above, no contraction (bitwise reproducible)
 *     lat_us[i] = max(1, ceil(t_s[i] * 1e6))
 * with the ctx's perf coefficients and caps.  F[i] (flops) and M[i] (bytes) as the cost model
 * gives them (App. A; exact integers).  t_s may be NULL.  Arrays: all device pointers or all host
 * pointers (host arrays are staged).  Errors: ASC_E_INVAL (NULL arrays, n < 0, mixed pointer
 * kinds), ASC_E_RANGE (some F[i] or M[i] >= 2^53: the int -> double conversion would round;
 * lat_us[i] = -1 there). */
asc_status asc_latency(asc_ctx* ctx, int64_t n, const uint64_t* F, const uint64_t* M, int64_t* lat_us,
                       double* t_s);

#ifdef __cplusplus
}
#endif
#endif
