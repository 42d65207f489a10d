/* oracle.h — CPU ORACLE (TEST INFRASTRUCTURE ONLY).
 *
 * A plain, slow, single-threaded-per-trace C++ transcription of Ascendra's
 * scheduler and batch-level simulator (arXiv 2504.20828, /root/reference/PAPER.md)
 * used to prove the CUDA path right.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  It shares no
 * code, header, table or constant generator with paper_2504_20828_b200/ or
 * include/asc.h; the two meet only through the seeded inputs of gen/.
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, Gnn = DESIGN.md reading.
 * Pins: see tests/test_oracle_*.py (every function below is pinned; none is
 * "parity unpinned" except where DESIGN.md §Pins says so).
 */
#ifndef ASC_ORACLE_H
#define ASC_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Model symbols of App. A.1; d = bytes per element (G10); tp divides h,n,m. */
typedef struct { int64_t h, n, s, n_kv, m, L, b, d, tp; } or_arch;
/* Regression coefficients C1..C5 and hardware caps F_H, M_H of Eq. 4-5. */
typedef struct { double c[5]; double F_H, M_H; } or_perf;
/* Instance partition, budgets and switches (readings G22-G41). */
typedef struct {
  int32_t n_lp, n_hp, bs, kv_lp, kv_hp, lp_max_batch, lp_tok, hp_tok;
  int32_t policy, offload, tickets, elastic, drop, hist_default;
  int64_t margin_us, delay_us;
  int32_t scheduler;  /* 0 Ascendra (LP/HP); 1 vLLM-like (G46); 2 Sarathi-like (G47) */
  int32_t chunk_tokens;  /* Sarathi-like per-batch token budget (decodes + prefill chunks, G47) */
  int32_t offload_rule;  /* 0 paper; 1 look-ahead: + prefill_us of the waiting requests
                            ahead in priority order (row f4, G50) */
  int32_t key_w[3];      /* policy 5 (WEIGHTED): key = w0 deadline + w1 prefill_us + w2 arrival */
} or_sched;

/* Eq. 1-3 with App. A.2/A.3 GEMM terms: exact integer F (flops) and M (bytes) of a batch of
 * np whole-prompt prefills p[] and nd decodes with contexts lhat[].  Returns 0, or 1 when a
 * result would reach 2^53 (not exactly representable in fp64). */
int or_cost(const or_arch* a, int32_t np, const int64_t* p, int32_t nd, const int64_t* lhat,
            uint64_t* F, uint64_t* M);
/* App. A.4 hybrid batch with chunked prefill, readings G48: nc chunks, chunk j has
 * l[j] prompt tokens already prefilled and processes c[j] more; plus nd decodes.  GEMM terms
 * count sum(c) + nd tokens; attention per head: chunk j costs M = 2 l s + 3 c s ceil(l/b) (its
 * cached context) + 2 c s + 3 c s ceil(c/b) (intra-chunk) and F = 2 s l c + 2 s c^2.
 * With every l = 0 this is or_cost of whole prompts c[].  Returns 0, or 1 at 2^53. */
int or_cost_chunked(const or_arch* a, int32_t nc, const int64_t* l, const int64_t* c, int32_t nd,
                    const int64_t* lhat, uint64_t* F, uint64_t* M);
/* Eq. 4-5: predicted seconds, fp64, fixed operation order, clamp at 0. */
double or_latency_s(const or_perf* pf, uint64_t F, uint64_t M);
/* G18/G17: integer microseconds = max(1, ceil(t * 1e6)). */
int64_t or_latency_us(const or_perf* pf, uint64_t F, uint64_t M);
/* or_latency_us (and, if t != NULL, or_latency_s) of n (F, M) pairs; a loop for the tests. */
void or_latency_n(const or_perf* pf, int64_t n, const uint64_t* F, const uint64_t* M,
                  int64_t* lat_us, double* t);
/* Convenience: latency of a batch in microseconds (or -1 on range error). */
int64_t or_batch_us(const or_arch* a, const or_perf* pf, int32_t np, const int64_t* p,
                    int32_t nd, const int64_t* lhat);

/* or_simulate_batch: trace_n_lp / trace_n_hp (may be NULL) give trace t its own subgroup
 * topology (row f3): n_lp >= 1, n_hp >= 0, n_lp + n_hp <= sc->n_lp + sc->n_hp.
 * req_key_offset_us (may be NULL): per-request value-function offset added to the key under
 * every policy (service classes; G51). */

/* Eq. 4-5 calibration ("perform a linear regression to find ... C1 ... C5", P:279
 * online refit; readings G49): for each of G groups of batch records (CSR off[],
 * exact F flops and M bytes, observed seconds y) the ridge least-squares coefficients
 *   c = argmin sum_i (x_i . c - y_i)^2 + lambda |c|^2,  x = (tM + tF, max(tM, tF), tM, tF, 1),
 * tM = M / M_H, tF = F / F_H, from the normal equations by Cholesky; coef[5g..5g+4] = C1..C5.
 * mean_err / max_err (may be NULL): in-sample mean and max of |pred - y| / y with pred the
 * Eq. 4-5 prediction of the fitted model (clamped at 0, or_latency_s).  Returns 0; 2 when a
 * group has fewer than 20 records or the regularised system is not positive definite. */
int or_fit_perf(const or_perf* pf, int32_t G, const int64_t* off, const uint64_t* F,
                const uint64_t* M, const double* y, double lambda, double* coef,
                double* mean_err, double* max_err);

/* Algorithm 1, literal: n requests with value val[] (higher = more urgent),
 * compute cost c[], memory cost mem[], token cost tok[]; budgets C, M, N plus the request-count
 * budget R (reading G22).  Writes the selected request indices in scan order; returns count. */
int32_t or_algorithm1(int32_t n, const int64_t* val, const int64_t* id, const int64_t* c,
                      const int64_t* mem, const int64_t* tok, int64_t C, int64_t M, int64_t N,
                      int64_t R, int32_t* selected);

/* Stateless LP decision over S segments (one LP formation without decode prep). */
int or_schedule_step(const or_arch* a, const or_perf* pf, const or_sched* sc, int32_t S,
                     const int64_t* seg_off, const int64_t* now_us, const int64_t* deadline_us,
                     const int32_t* eff_prompt, const uint8_t* flags, const int32_t* dec_count,
                     const int64_t* dec_ctx_sum, const int64_t* tbt_slo_us,
                     const int32_t* budget_tokens, const int32_t* budget_blocks,
                     const int32_t* budget_reqs,
                     int32_t* admit_idx, int32_t* admit_cnt, int32_t* offload_idx,
                     int32_t* offload_cnt, int32_t* drop_idx, int32_t* drop_cnt,
                     int64_t* batch_lat_us, int32_t* prefill_us);

/* Full batch-level simulation of T independent traces (CSR), threads across traces. */
int or_simulate_batch(const or_arch* a, const or_perf* pf, const or_sched* sc, int32_t T,
                      const int64_t* trace_off, const int64_t* arrival_us,
                      const int32_t* prompt_len, const int32_t* output_len,
                      const int64_t* ttft_slo_us, const int64_t* tbt_slo_us,
                      const int64_t* req_ttft_slo_us,
                      const int32_t* trace_n_lp, const int32_t* trace_n_hp,
                      const int64_t* req_key_offset_us,
                      int64_t* first_token_us, int64_t* done_us, int64_t* prefill_start_us,
                      uint32_t* status, uint64_t* digest, int64_t* decisions,
                      int64_t* evaluations, int32_t nthreads, int32_t check_invariants);

/* Goodput numerator/denominator per trace. Returns 0, or 5 if a trace is empty. */
int or_goodput(int32_t T, const int64_t* trace_off, const int64_t* arrival_us,
               const int32_t* output_len, const int64_t* ttft_slo_us, const int64_t* tbt_slo_us,
               const int64_t* req_ttft_slo_us, const int64_t* first_token_us,
               const int64_t* done_us, const uint32_t* status, uint64_t* good, uint64_t* total);

/* Outcome summary per trace (row a8; Fig. 10 metric set; SPEC S:543-590 metrics module;
 * DESIGN.md reading G52).  Every output array [T] may be NULL.
 *   completed / dropped         requests in state COMPLETED / DROPPED
 *   violating                   completed but not good (TTFT or mean-TBT SLO missed)
 *   tokens                      sum of output_len over completed requests (dropped contribute 0)
 *   ttft_p{50,90,99}_us         nearest-rank percentile (the ceil(q n / 100)-th smallest)
 *                               of first_token - arrival over requests with a first token; -1 if none
 *   tbt_sum_us / tbt_tokens     sum of (done - first) and of (output_len - 1) over completed
 *                               requests with output_len > 1 (mean TBT = tbt_sum_us / tbt_tokens)
 *   delay_sum_{lp,hp}_us / delay_cnt_{lp,hp}
 *                               scheduling delay prefill_start - arrival summed over
 *                               requests with a prefill start, split by the type of the serving
 *                               instance (index < n_lp of the trace = LP)
 *   last_done_us                latest done_us of the trace (-1 if none completed)
 * trace_n_lp: per-trace LP count (may be NULL: n_lp for every trace).  Returns 0. */
int or_summarize(int32_t T, const int64_t* trace_off, const int64_t* arrival_us,
                 const int32_t* output_len, const int64_t* ttft_slo_us, const int64_t* tbt_slo_us,
                 const int64_t* req_ttft_slo_us, const int32_t* trace_n_lp, int32_t n_lp,
                 const int64_t* first_token_us, const int64_t* done_us,
                 const int64_t* prefill_start_us, const uint32_t* status,
                 int64_t* completed, int64_t* dropped, int64_t* violating, int64_t* tokens,
                 int64_t* ttft_p50_us, int64_t* ttft_p90_us, int64_t* ttft_p99_us,
                 int64_t* tbt_sum_us, int64_t* tbt_tokens,
                 int64_t* delay_sum_lp_us, int64_t* delay_cnt_lp,
                 int64_t* delay_sum_hp_us, int64_t* delay_cnt_hp, int64_t* last_done_us);

const char* or_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
