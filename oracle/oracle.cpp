// oracle.cpp — CPU ORACLE (TEST INFRASTRUCTURE ONLY; see oracle.h).
//
// Plain transcription of PAPER.md §5-§6 and Appendix A, in the paper's order and
// notation, with the DESIGN.md readings (Gnn) where the paper is silent.  No
// blocking, fusion or incremental data structures: every formation re-annotates,
// re-sorts and re-scans its queue exactly as Algorithm 1 states.  Built with
// -ffp-contract=off so every fp64 operation is a separate IEEE-754 RN operation.
#include "oracle.h"

#include <algorithm>
#include <map>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

static thread_local std::string g_err;
static void set_err(const std::string& s) { g_err = s; }
extern "C" const char* or_last_error(void) { return g_err.c_str(); }

static const uint64_t TWO53 = 1ull << 53;
static const int64_t INF64 = INT64_MAX;

static int64_t ceil_div(int64_t x, int64_t y) { return (x + y - 1) / y; }

// --------------------------------------------------------------------------------------------
// Cost model: Eq. 1, Eq. 2, Eq. 3, Tables 3-4,
// Eq. 6, Eq. 7, readings G1-G12.  Per layer, then x L (G11), memory
// counted in elements then x d bytes (G10).  GEMM weight terms 4h^2 + 2hm counted once per
// non-empty batch (G8).
// --------------------------------------------------------------------------------------------
extern "C" int or_cost(const or_arch* a, int32_t np, const int64_t* p, int32_t nd,
                       const int64_t* lhat, uint64_t* F, uint64_t* M) {
  const uint64_t h = a->h, n = a->n, s = a->s, m = a->m, b = a->b, L = a->L, d = a->d;
  // t = number of tokens that pass through the GEMMs (prefill tokens + one per decode).
  uint64_t t = 0;
  for (int32_t i = 0; i < np; i++) t += (uint64_t)p[i];
  const uint64_t tok = t + (uint64_t)nd;
  const uint64_t G = (np + nd) > 0 ? 1 : 0;
  // Table 3 + Table 4 rows: QKV 3 t h^2, out t h^2, FFN in t h m, FFN out t h m.
  const uint64_t gemm_F = 3 * tok * h * h + tok * h * h + tok * h * m + tok * h * m;
  // Memory read + write of the same rows: (th + 3h^2) + 3th, (th + h^2) + th,
  // (th + hm) + tm, (tm + hm) + th  =  8th + 4h^2 + 2hm + 2tm with weights once (G8).
  const uint64_t gemm_M = G * (3 * h * h + h * h + h * m + h * m) +
                          (tok * h + 3 * tok * h) + (tok * h + tok * h) +
                          (tok * h + tok * m) + (tok * m + tok * h);
  // Eq. 1: per head, M_p = sum 2 l_i s + 3 l_i s ceil(l_i / b) (G9), F_p = sum 2 s l_i^2.
  uint64_t Mp = 0, Fp = 0;
  for (int32_t i = 0; i < np; i++) {
    const uint64_t li = (uint64_t)p[i];
    Mp += 2 * li * s + 3 * li * s * (uint64_t)ceil_div((int64_t)li, (int64_t)b);
    Fp += 2 * s * li * li;
  }
  // Eq. 2 with the +2s inside the sum (G3): M_d = sum 2 lhat_i s + 2 s, F_d = sum 2 lhat_i s.
  uint64_t Md = 0, Fd = 0;
  for (int32_t j = 0; j < nd; j++) {
    const uint64_t lj = (uint64_t)lhat[j];
    Md += 2 * lj * s + 2 * s;
    Fd += 2 * lj * s;
  }
  // Eq. 3: one decoding layer M = (M_p + M_d) n + M(GEMM), F = (F_p + F_d) n + F(GEMM).
  const uint64_t M_layer = (Mp + Md) * n + gemm_M;
  const uint64_t F_layer = (Fp + Fd) * n + gemm_F;
  *F = L * F_layer;
  *M = L * M_layer * d;
  // uint64 wrap guard: the same sums in fp64; far above 2^53 means out of range, whatever the
  // wrapped integers say (every term is a product of non-negative integers)
  double fF = 0, fM = 0;
  for (int32_t i = 0; i < np; i++) {
    const double li = (double)p[i];
    fM += 2 * li * s + 3 * li * s * (double)ceil_div(p[i], (int64_t)b);
    fF += 2 * (double)s * li * li;
  }
  for (int32_t j = 0; j < nd; j++) { fM += 2 * (double)lhat[j] * s + 2.0 * s; fF += 2 * (double)lhat[j] * s; }
  const double ft = (double)t + (double)nd;
  fF = (double)L * (fF * (double)n + ft * (4.0 * h * h + 2.0 * h * m));
  fM = (double)L * (double)d * (fM * (double)n + (double)G * (4.0 * h * h + 2.0 * h * m) + ft * (8.0 * h + 2.0 * m));
  if (fF >= 0x1p62 || fM >= 0x1p62) return 1;
  return (*F >= TWO53 || *M >= TWO53) ? 1 : 0;
}

// App. A.4 hybrid batch with chunked prefill, readings G48.  M_m's garbled
// "8 sum l_i h + 2 sum l_i m" activations are the chunk tokens c_i (the GEMM rows this batch
// processes, as in Tables 3-4); "l_i / b" is ceil(l_i / b) (G9); the chunk's self-attention
// (absent from A.4, whose terms vanish at l_i = 0) is Eq. 1 applied to the chunk, so
// whole prompts (l = 0) cost exactly what or_cost charges.  Same per-layer / x L / x d rules.
extern "C" int or_cost_chunked(const or_arch* a, int32_t nc, const int64_t* l, const int64_t* c,
                               int32_t nd, const int64_t* lhat, uint64_t* F, uint64_t* M) {
  const uint64_t h = a->h, n = a->n, s = a->s, m = a->m, b = a->b, L = a->L, d = a->d;
  uint64_t t = 0;
  for (int32_t i = 0; i < nc; i++) t += (uint64_t)c[i];
  const uint64_t tok = t + (uint64_t)nd;
  const uint64_t G = (nc + nd) > 0 ? 1 : 0;
  const uint64_t gemm_F = 3 * tok * h * h + tok * h * h + tok * h * m + tok * h * m;
  const uint64_t gemm_M = G * (3 * h * h + h * h + h * m + h * m) +
                          (tok * h + 3 * tok * h) + (tok * h + tok * h) +
                          (tok * h + tok * m) + (tok * m + tok * h);
  uint64_t Mp = 0, Fp = 0;
  for (int32_t i = 0; i < nc; i++) {
    const uint64_t li = (uint64_t)l[i], ci = (uint64_t)c[i];
    // cached context of the chunk: 2 l s (load k, v) + 3 c s per k/v block (q, o read/write)
    Mp += 2 * li * s + 3 * ci * s * (uint64_t)ceil_div((int64_t)li, (int64_t)b);
    Fp += 2 * s * li * ci;
    // the chunk's own tokens (Eq. 1 on the chunk)
    Mp += 2 * ci * s + 3 * ci * s * (uint64_t)ceil_div((int64_t)ci, (int64_t)b);
    Fp += 2 * s * ci * ci;
  }
  uint64_t Md = 0, Fd = 0;
  for (int32_t j = 0; j < nd; j++) {
    const uint64_t lj = (uint64_t)lhat[j];
    Md += 2 * lj * s + 2 * s;
    Fd += 2 * lj * s;
  }
  const uint64_t M_layer = (Mp + Md) * n + gemm_M;
  const uint64_t F_layer = (Fp + Fd) * n + gemm_F;
  *F = L * F_layer;
  *M = L * M_layer * d;
  return (*F >= TWO53 || *M >= TWO53) ? 1 : 0;
}

// Eq. 4-5: t = C1 (tM + tF) + C2 max(tM, tF) + C3 tM + C4 tF + C5,
// tM = M / M_H, tF = F / F_H.  Fixed left-to-right order; clamp negative to 0 (G17).
extern "C" double or_latency_s(const or_perf* pf, uint64_t F, uint64_t M) {
  const double tM = (double)M / pf->M_H;
  const double tF = (double)F / pf->F_H;
  const double mx = (tM > tF) ? tM : tF;
  double t = pf->c[0] * (tM + tF);
  t = t + pf->c[1] * mx;
  t = t + pf->c[2] * tM;
  t = t + pf->c[3] * tF;
  t = t + pf->c[4];
  if (!(t > 0.0)) t = 0.0;
  return t;
}

// Eq. 4-5 calibration (G49).  Plain: features per record, the 5x5
// Gram matrix and X'y by sequential sums in record order, + lambda on the diagonal, Cholesky
// A = L L', forward and back substitution.  In-sample error through or_latency_s itself.
extern "C" int or_fit_perf(const or_perf* pf, int32_t G, const int64_t* off, const uint64_t* F,
                           const uint64_t* M, const double* y, double lambda, double* coef,
                           double* mean_err, double* max_err) {
  for (int32_t g = 0; g < G; g++) {
    const int64_t lo = off[g], hi = off[g + 1];
    if (hi - lo < 20) { set_err("fit: a group has fewer than 20 records (S:154)"); return 2; }
    double A[5][5] = {{0}}, b[5] = {0};
    for (int64_t i = lo; i < hi; i++)
      if (!(y[i] > 0.0 && y[i] < HUGE_VAL)) { set_err("fit: observed latency must be > 0"); return 1; }
    for (int64_t i = lo; i < hi; i++) {
      const double tM = (double)M[i] / pf->M_H;
      const double tF = (double)F[i] / pf->F_H;
      const double x[5] = {tM + tF, tM > tF ? tM : tF, tM, tF, 1.0};
      for (int j = 0; j < 5; j++) {
        for (int k = j; k < 5; k++) A[j][k] = A[j][k] + x[j] * x[k];
        b[j] = b[j] + x[j] * y[i];
      }
    }
    for (int j = 0; j < 5; j++) {
      A[j][j] = A[j][j] + lambda;
      for (int k = 0; k < j; k++) A[j][k] = A[k][j];
    }
    // Cholesky: L[j][j] = sqrt(A[j][j] - sum_k L[j][k]^2), L[i][j] = (A[i][j] - sum_k L[i][k] L[j][k]) / L[j][j]
    double Lc[5][5] = {{0}};
    for (int j = 0; j < 5; j++) {
      double d = A[j][j];
      for (int k = 0; k < j; k++) d = d - Lc[j][k] * Lc[j][k];
      if (!(d > 0.0)) { set_err("fit: regularised normal equations not positive definite"); return 2; }
      Lc[j][j] = std::sqrt(d);
      for (int i = j + 1; i < 5; i++) {
        double v = A[i][j];
        for (int k = 0; k < j; k++) v = v - Lc[i][k] * Lc[j][k];
        Lc[i][j] = v / Lc[j][j];
      }
    }
    double z[5], c[5];
    for (int i = 0; i < 5; i++) {  // L z = b
      double v = b[i];
      for (int k = 0; k < i; k++) v = v - Lc[i][k] * z[k];
      z[i] = v / Lc[i][i];
    }
    for (int i = 4; i >= 0; i--) {  // L' c = z
      double v = z[i];
      for (int k = i + 1; k < 5; k++) v = v - Lc[k][i] * c[k];
      c[i] = v / Lc[i][i];
    }
    for (int j = 0; j < 5; j++) coef[5 * g + j] = c[j];
    if (mean_err || max_err) {
      or_perf fitted = *pf;
      for (int j = 0; j < 5; j++) fitted.c[j] = c[j];
      double sum = 0.0, mx = 0.0;
      for (int64_t i = lo; i < hi; i++) {
        const double pred = or_latency_s(&fitted, F[i], M[i]);
        const double e = std::fabs(pred - y[i]) / y[i];
        sum = sum + e;
        if (e > mx) mx = e;
      }
      if (mean_err) mean_err[g] = sum / (double)(hi - lo);
      if (max_err) max_err[g] = mx;
    }
  }
  return 0;
}

// G18: continuous seconds -> event time in integer microseconds, at least 1 (G17).
extern "C" int64_t or_latency_us(const or_perf* pf, uint64_t F, uint64_t M) {
  const double t = or_latency_s(pf, F, M);
  const double us = std::ceil(t * 1e6);
  int64_t v = (int64_t)us;
  return v < 1 ? 1 : v;
}

// Test convenience: or_latency_s / or_latency_us over n (F, M) pairs (a plain loop; no new
// arithmetic).  t may be NULL.
extern "C" void or_latency_n(const or_perf* pf, int64_t n, const uint64_t* F, const uint64_t* M,
                             int64_t* lat_us, double* t) {
  for (int64_t i = 0; i < n; i++) {
    lat_us[i] = or_latency_us(pf, F[i], M[i]);
    if (t) t[i] = or_latency_s(pf, F[i], M[i]);
  }
}

extern "C" int64_t or_batch_us(const or_arch* a, const or_perf* pf, int32_t np,
                               const int64_t* p, int32_t nd, const int64_t* lhat) {
  uint64_t F, M;
  if (or_cost(a, np, p, nd, lhat, &F, &M)) return -1;
  return or_latency_us(pf, F, M);
}

static int64_t prefill_us_of(const or_arch* a, const or_perf* pf, int64_t p) {
  return or_batch_us(a, pf, 1, &p, 0, nullptr);
}

// --------------------------------------------------------------------------------------------
// Algorithm 1 "Out Of Order Scheduling", line by line.  Ties in line 3 are broken by
// ascending id (G20).  R (request-count budget, G22) joins line 7's test.
// --------------------------------------------------------------------------------------------
extern "C" int32_t or_algorithm1(int32_t n, const int64_t* val, const int64_t* id,
                                 const int64_t* c, const int64_t* mem, const int64_t* tok,
                                 int64_t C, int64_t M, int64_t N, int64_t R, int32_t* selected) {
  // lines 1-2: annotate (done by the caller: val, c, mem, tok)
  std::vector<int32_t> W(n);
  for (int32_t i = 0; i < n; i++) W[i] = i;
  // line 3: sort W by val descending (ties: ascending id)
  std::sort(W.begin(), W.end(), [&](int32_t x, int32_t y) {
    if (val[x] != val[y]) return val[x] > val[y];
    return id[x] < id[y];
  });
  int32_t k = 0;  // line 4: selected_items <- []
  for (int32_t q = 0; q < n; q++) {          // line 5
    const int32_t w = W[q];
    if (C > 0 && M > 0 && N > 0) {             // line 6
      if (C > c[w] && M > mem[w] && N > tok[w] && R >= 1) {  // line 7
        selected[k++] = w;                     // line 8
        if (C != INF64) C = C - c[w];          // line 9 (C = +inf when no decodes, G22)
        M = M - mem[w];                        // line 10
        N = N - tok[w];                        // line 11
        R = R - 1;
      } else {
        break;                                 // lines 12-13
      }
    }
  }
  return k;  // line 14
}

// Priority value pi (G19): Algorithm 1 sorts by val descending; we use val = -key.
// EDF_LAXITY key = deadline - prefill_us; EDF_DEADLINE key = deadline; SJF key = prefill_us;
// LJF key = -prefill_us; FCFS key = arrival.
static int64_t key_of(int policy, int64_t arrival, int64_t deadline, int64_t pf_us,
                      const int32_t* w = nullptr) {
  switch (policy) {
    case 0: return deadline - pf_us;
    case 1: return deadline;
    case 2: return pf_us;
    case 3: return -pf_us;
    case 5: return (int64_t)w[0] * deadline + (int64_t)w[1] * pf_us + (int64_t)w[2] * arrival;
    default: return arrival;
  }
}

static void apply_tp(const or_arch* in, or_arch* out) {
  *out = *in;
  if (in->tp > 1) { out->h /= in->tp; out->n /= in->tp; out->m /= in->tp; out->n_kv /= in->tp; }
}

static bool check_cfg(const or_arch* a, const or_perf* pf) {
  if (a->h <= 0 || a->n <= 0 || a->s <= 0 || a->m <= 0 || a->L <= 0 || a->b <= 0 || a->d <= 0 ||
      a->tp <= 0) { set_err("arch: non-positive field"); return false; }
  if (a->h != a->n * a->s) { set_err("arch: h != n*s"); return false; }
  if (a->h % a->tp || a->n % a->tp || a->m % a->tp) { set_err("arch: tp does not divide"); return false; }
  if (!(pf->F_H > 0) || !(pf->M_H > 0)) { set_err("perf: F_H/M_H must be > 0"); return false; }
  return true;
}

// --------------------------------------------------------------------------------------------
// Stateless LP decision (one formation of §5 without decode preparation).
// --------------------------------------------------------------------------------------------
extern "C" int or_schedule_step(const or_arch* a_in, const or_perf* pf, const or_sched* sc,
                                int32_t S, const int64_t* seg_off, const int64_t* now_us,
                                const int64_t* deadline_us, const int32_t* eff_prompt,
                                const uint8_t* flags, const int32_t* dec_count,
                                const int64_t* dec_ctx_sum, const int64_t* tbt_slo_us,
                                const int32_t* budget_tokens, const int32_t* budget_blocks,
                                const int32_t* budget_reqs, int32_t* admit_idx,
                                int32_t* admit_cnt, int32_t* offload_idx, int32_t* offload_cnt,
                                int32_t* drop_idx, int32_t* drop_cnt, int64_t* batch_lat_us,
                                int32_t* prefill_us) {
  if (sc->policy == 5 || sc->offload_rule != 0) { set_err("step: WEIGHTED policy / look-ahead offload are simulator-only"); return 2; }
  if (!check_cfg(a_in, pf)) return 2;
  or_arch a;
  apply_tp(a_in, &a);
  int64_t Whp = 0;
  if (sc->offload && sc->n_hp >= 1) {
    Whp = prefill_us_of(&a, pf, sc->hp_tok);  // worst-case HP batch (G24)
    if (Whp < 0) { set_err("range: W_hp"); return 6; }
  }
  for (int32_t sg = 0; sg < S; sg++) {
    const int64_t lo = seg_off[sg], hi = seg_off[sg + 1];
    const int64_t now = now_us[sg];
    const int32_t n = (int32_t)(hi - lo);
    std::vector<int64_t> pfu(n), blk(n), tok(n), key(n), dl(n), id(n), val(n);
    std::vector<bool> dropped(n, false);
    for (int32_t i = 0; i < n; i++) {
      const int64_t e = lo + i;
      if (eff_prompt[e] < 1) { set_err("eff_prompt < 1"); return 1; }
      if (eff_prompt[e] >= (1 << 24)) { set_err("range: eff_prompt >= 2^24"); return 6; }
      pfu[i] = prefill_us_of(&a, pf, eff_prompt[e]);
      if (pfu[i] < 0) { set_err("range: prefill cost"); return 6; }
      if (prefill_us) prefill_us[e] = (int32_t)pfu[i];
      blk[i] = ceil_div((int64_t)eff_prompt[e] + 1, sc->bs);   // G23 / S:412
      tok[i] = eff_prompt[e];
      dl[i] = deadline_us[e];
      id[i] = i;
      key[i] = key_of(sc->policy, 0 /* entries are in arrival order: FCFS = position */,
                      dl[i], pfu[i]);
      val[i] = -key[i];
      const bool ever = flags[e] & 1;
      // drop rule (G34): waiting, never prefilled, strictly past its deadline
      if (sc->drop && !ever && now > dl[i]) dropped[i] = true;
    }
    // TBT residual C (G22): tbt - decode-only latency, +inf without decodes.
    int64_t C = INF64;
    const int32_t Bd = dec_count[sg];
    if (Bd > 0) {
      // Eq. 2 depends on the contexts only through their sum: materialise contexts with that sum.
      std::vector<int64_t> lh(Bd, 1);
      lh[0] = dec_ctx_sum[sg] - (Bd - 1);
      if (lh[0] < 1) { set_err("dec_ctx_sum < dec_count"); return 1; }
      const int64_t dus = or_batch_us(&a, pf, 0, nullptr, Bd, lh.data());
      if (dus < 0) { set_err("range: decode cost"); return 6; }
      C = tbt_slo_us[sg] - dus;
    }
    // Algorithm 1 over the non-dropped entries.
    std::vector<int32_t> live;
    for (int32_t i = 0; i < n; i++) if (!dropped[i]) live.push_back(i);
    const int32_t nl = (int32_t)live.size();
    std::vector<int64_t> v2(nl), id2(nl), c2(nl), m2(nl), t2(nl);
    for (int32_t q = 0; q < nl; q++) {
      v2[q] = val[live[q]]; id2[q] = id[live[q]]; c2[q] = pfu[live[q]];
      m2[q] = blk[live[q]]; t2[q] = tok[live[q]];
    }
    std::vector<int32_t> sel(nl > 0 ? nl : 1);
    const int32_t k = or_algorithm1(nl, v2.data(), id2.data(), c2.data(), m2.data(), t2.data(),
                                    C, budget_blocks[sg], budget_tokens[sg], budget_reqs[sg],
                                    sel.data());
    std::vector<bool> admitted(n, false);
    std::vector<int64_t> ap;
    for (int32_t j = 0; j < k; j++) {
      const int32_t i = live[sel[j]];
      admitted[i] = true;
      admit_idx[lo + j] = (int32_t)(lo + i);
      ap.push_back(tok[i]);
    }
    admit_cnt[sg] = k;
    // Offload (§5.3, G24): non-admitted, never prefilled, not on HP, ascending id.
    int32_t no = 0, ndp = 0;
    for (int32_t i = 0; i < n; i++) {
      const int64_t e = lo + i;
      if (dropped[i]) { drop_idx[lo + ndp++] = (int32_t)e; continue; }
      if (!(sc->offload && sc->n_hp >= 1) || admitted[i]) continue;
      const bool ever = flags[e] & 1, onhp = flags[e] & 2;
      if (!ever && !onhp && dl[i] - now <= pfu[i] + Whp + sc->margin_us)
        offload_idx[lo + no++] = (int32_t)e;
    }
    offload_cnt[sg] = no;
    drop_cnt[sg] = ndp;
    // Batch latency of the formed hybrid batch (§5.4, Eq. 3-5).
    if (k > 0 || Bd > 0) {
      std::vector<int64_t> lh;
      if (Bd > 0) { lh.assign(Bd, 1); lh[0] = dec_ctx_sum[sg] - (Bd - 1); }
      const int64_t us = or_batch_us(&a, pf, k, ap.data(), Bd, lh.data());
      if (us < 0) { set_err("range: batch cost"); return 6; }
      batch_lat_us[sg] = us;
    } else {
      batch_lat_us[sg] = 0;
    }
  }
  return 0;
}

// --------------------------------------------------------------------------------------------
// Batch-level discrete-event simulation of one trace (§4-§6, canonical phases of DESIGN.md).
// --------------------------------------------------------------------------------------------
namespace {

uint64_t mix(uint64_t x) {  // splitmix64 finalizer (digest only)
  uint64_t z = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

enum { UNFINISHED = 0, COMPLETED = 1, DROPPED = 2 };

struct Req {
  int64_t arrival, ttft, deadline;
  int64_t p, o;        // prompt and output lengths
  int64_t g = 0;       // tokens generated so far
  int64_t eff;         // effective prompt (prompt + generated after preemption)
  int64_t held = 0;    // KV blocks held
  int64_t cdone = 0;   // prompt tokens already prefilled (Sarathi-like chunks, G47)
  int64_t koff = 0;    // value-function offset of the request's service class (G51)
  bool ever = false, onhp = false, ticketed = false, offloaded = false;
  int state = UNFINISHED;
  int64_t first = -1, done = -1, pstart = -1;
  int inst = 255;
  int64_t npre = 0;
};

struct Inst {
  bool hp;
  std::vector<int> waiting;   // LP: arrival/insertion order; HP: FCFS by (arrival, id)
  std::vector<int> D;         // decoding set
  int64_t kv_total, kv_free;
  bool busy = false;
  int64_t end = 0;
  std::vector<int> batch_pf;  // prefills of the running batch
  bool batch_dec = false;     // did the running batch include the decode set?
  bool ticket = false;
  int tk_live = 0;            // resident ticketed requests (at most one, G29)
  int64_t hist_sum = 0, hist_cnt = 0;
  uint64_t hash = 0;
  uint64_t nrec = 0;  // recorded formations (digest position)
};

struct Sim {
  const or_arch* a;
  const or_perf* pf;
  const or_sched* sc;
  std::vector<Req> r;
  std::vector<Inst> I;
  int64_t tbt;
  int64_t Whp = 0;
  int rr_lp = 0, rr_hp = 0;
  struct Flight { int64_t t; int req; int hp; };
  std::vector<Flight> inflight;
  int64_t decisions = 0, evaluations = 0;
  bool check;
  std::string err;

  int64_t pf_us(int64_t eff) { return prefill_us_of(a, pf, eff); }
  int64_t blk(int64_t eff) { return ceil_div(eff + 1, sc->bs); }
  int64_t key(int i) {  // value function (G19) + the request's class offset (G51)
    return key_of(sc->policy, r[i].arrival, r[i].deadline, pf_us(r[i].eff), sc->key_w) + r[i].koff;
  }
  bool fcfs_less(int x, int y) {
    if (r[x].arrival != r[y].arrival) return r[x].arrival < r[y].arrival;
    return x < y;
  }
  void hp_insert(Inst& h, int i) {
    h.waiting.push_back(i);
    std::sort(h.waiting.begin(), h.waiting.end(), [&](int x, int y) { return fcfs_less(x, y); });
  }
  // Digest: the record of one formation hashes as rec = sum_i mix(v_i + (i+1) * G)
  // (mod 2^64; position-keyed, so order-sensitive); the instance digest is the sum over its
  // recorded formations f = 0, 1, ... of mix(rec_f + (f+1) * G2) (formation-index keyed).
  void record(Inst& in, const std::vector<uint64_t>& v) {
    uint64_t rec = 0;
    for (size_t i = 0; i < v.size(); i++) rec += mix(v[i] + (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull);
    in.nrec += 1;
    in.hash += mix(rec + (uint64_t)in.nrec * 0xD1B54A32D192ED03ull);
  }
  int64_t lat(const std::vector<int>& pre, const std::vector<int>& dec) {
    std::vector<int64_t> p, l;
    for (int i : pre) p.push_back(r[i].eff);
    for (int j : dec) l.push_back(r[j].p + r[j].g);  // lhat = prompt + generated
    const int64_t us = or_batch_us(a, pf, (int32_t)p.size(), p.data(), (int32_t)l.size(),
                                   l.data());
    if (us < 0 && err.empty()) err = "range: batch cost reaches 2^53";
    return us;
  }

  void finish(Inst& in, int i, int64_t T) {
    r[i].state = COMPLETED;
    r[i].done = T;
    in.kv_free += r[i].held;
    r[i].held = 0;
    if (in.hp && r[i].ticketed) in.tk_live -= 1;
    if (in.hp) { in.hist_sum += r[i].o; in.hist_cnt += 1; }  // decode-length history
  }

  // Phase A: the running batch of instance k ends at T.
  void complete(int k, int64_t T) {
    Inst& in = I[k];
    std::vector<int> keep;
    if (in.batch_dec) {
      for (int j : in.D) {
        r[j].g += 1;
        if (r[j].g == r[j].o) finish(in, j, T); else keep.push_back(j);
      }
      in.D = keep;
    }
    for (int i : in.batch_pf) {
      if (sc->scheduler == 2) {
        if (r[i].cdone < r[i].eff) continue;  // partial chunk: stays at the head of the queue
        in.waiting.erase(std::find(in.waiting.begin(), in.waiting.end(), i));
      }
      r[i].g += 1;
      if (r[i].first < 0) r[i].first = T;  // TTFT: first token at the end of its prefill
      if (r[i].g == r[i].o) finish(in, i, T); else in.D.push_back(i);
    }
    in.batch_pf.clear();
    in.batch_dec = false;
    in.busy = false;
  }

  // Controller routing (G29-G30).
  void route(int i) {
    if (sc->tickets) {
      for (int h = sc->n_lp; h < (int)I.size(); h++) {
        if (I[h].ticket) {
          I[h].ticket = false;
          I[h].tk_live += 1;
          r[i].ticketed = true;
          r[i].onhp = true;
          hp_insert(I[h], i);
          return;
        }
      }
    }
    I[rr_lp].waiting.push_back(i);
    rr_lp = (rr_lp + 1) % sc->n_lp;
  }

  std::vector<int> drop_step(Inst& in, int64_t T) {
    std::vector<int> dropped, keep;
    for (int i : in.waiting) {
      if (sc->drop && !r[i].ever && T > r[i].deadline) {  // P:614, G34
        r[i].state = DROPPED;
        if (in.hp && r[i].ticketed) in.tk_live -= 1;
        dropped.push_back(i);
      } else {
        keep.push_back(i);
      }
    }
    in.waiting = keep;
    std::sort(dropped.begin(), dropped.end());
    return dropped;
  }

  // Decode preparation with preemption by recomputation (G31).
  std::vector<int> decode_prep(Inst& in) {
    std::vector<int> pre;
    auto need_of = [&](int j) { return ceil_div(r[j].p + r[j].g, sc->bs) - r[j].held; };
    int64_t need = 0;
    for (int j : in.D) need += need_of(j);
    while (need > in.kv_free) {
      int v = in.D[0];
      for (int j : in.D)
        if (r[j].arrival > r[v].arrival || (r[j].arrival == r[v].arrival && j > v)) v = j;
      need -= need_of(v);
      in.kv_free += r[v].held;
      r[v].held = 0;
      in.D.erase(std::find(in.D.begin(), in.D.end(), v));
      r[v].eff = r[v].p + r[v].g;  // append generated tokens to the prompt
      r[v].cdone = 0;
      r[v].npre += 1;
      pre.push_back(v);
      if (in.hp) hp_insert(in, v); else in.waiting.push_back(v);
    }
    for (int j : in.D) {
      const int64_t gr = need_of(j);
      r[j].held += gr;
      in.kv_free -= gr;
    }
    return pre;
  }

  void admit(Inst& in, int k, int i, int64_t T) {
    r[i].ever = true;
    if (r[i].pstart < 0) r[i].pstart = T;
    const int64_t b = blk(r[i].eff);
    r[i].held = b;
    in.kv_free -= b;
    r[i].inst = k;
    in.waiting.erase(std::find(in.waiting.begin(), in.waiting.end(), i));
  }

  void form_lp(int k, int64_t T) {
    Inst& in = I[k];
    std::vector<int> dropped = drop_step(in, T);
    std::vector<int> pre = decode_prep(in);
    evaluations += (int64_t)in.waiting.size();
    // Budgets (G22): N tokens, M free blocks, R = batch cap - decodes, C = TBT residual.
    const int64_t N = sc->lp_tok, M = in.kv_free, R = sc->lp_max_batch - (int64_t)in.D.size();
    int64_t C = INF64;
    if (!in.D.empty()) C = tbt - lat({}, in.D);
    // Algorithm 1 lines 1-2: annotate every waiting request with val, C, M, prefill tokens.
    const int n = (int)in.waiting.size();
    std::vector<int64_t> val(n), id(n), c(n), mem(n), tok(n);
    for (int q = 0; q < n; q++) {
      const int i = in.waiting[q];
      val[q] = -key(i);
      id[q] = i;
      c[q] = pf_us(r[i].eff);
      mem[q] = blk(r[i].eff);
      tok[q] = r[i].eff;
    }
    std::vector<int32_t> sel(n > 0 ? n : 1);
    const int32_t ks = or_algorithm1(n, val.data(), id.data(), c.data(), mem.data(), tok.data(),
                                     C, M, N, R, sel.data());
    std::vector<int> adm;
    for (int32_t j = 0; j < ks; j++) adm.push_back(in.waiting[sel[j]]);
    for (int i : adm) admit(in, k, i, T);
    // Offload (§5.3, G24): remaining never-prefilled requests projected to miss TTFT.
    std::vector<int> off;
    if (sc->offload && sc->n_hp >= 1) {
      // look-ahead (G50): the prefill time of every waiting request ahead in priority order
      std::map<int, int64_t> ahead;
      if (sc->offload_rule == 1) {
        std::vector<int> ord = in.waiting;
        std::sort(ord.begin(), ord.end(), [&](int x, int y) {
          const int64_t kx = key(x), ky = key(y);
          return kx != ky ? kx < ky : x < y;
        });
        int64_t sum = 0;
        for (int i : ord) { ahead[i] = sum; sum += pf_us(r[i].eff); }
      }
      std::vector<int> ids = in.waiting;
      std::sort(ids.begin(), ids.end());
      for (int i : ids)
        if (!r[i].ever && !r[i].onhp &&
            r[i].deadline - T <= pf_us(r[i].eff) + Whp + sc->margin_us + (sc->offload_rule == 1 ? ahead[i] : 0))
          off.push_back(i);
      for (int i : off) {
        in.waiting.erase(std::find(in.waiting.begin(), in.waiting.end(), i));
        r[i].onhp = true;
        r[i].offloaded = true;
        const int h = sc->n_lp + rr_hp;
        rr_hp = (rr_hp + 1) % sc->n_hp;
        if (sc->delay_us == 0) hp_insert(I[h], i);
        else inflight.push_back({T + sc->delay_us, i, h});
      }
    }
    // Batch (§5.4): decodes piggybacked with the admitted prefills.
    const bool nonempty = !adm.empty() || !in.D.empty();
    int64_t l = 0;
    if (nonempty) {
      l = lat(adm, in.D);
      in.busy = true;
      in.end = T + l;
      in.batch_pf = adm;
      in.batch_dec = !in.D.empty();
      decisions++;
    }
    if (nonempty || !off.empty() || !dropped.empty() || !pre.empty())
      log(in, T, k, adm, nonempty ? (int64_t)in.D.size() : 0, off, dropped, pre, l);
  }

  bool hp_prefill(Inst& in, int k, int64_t T, std::vector<int>& adm) {
    // FCFS (G26) under the token limit, elastic when enabled (G28).
    int64_t limit = sc->hp_tok;
    if (sc->elastic) {
      const int64_t mean = in.hist_cnt ? in.hist_sum / in.hist_cnt : sc->hist_default;
      const int64_t avail = in.kv_free * sc->bs - mean * ((int64_t)in.D.size() + 1);
      if (10 * avail > in.kv_total * sc->bs) limit = sc->hp_tok + avail;
    }
    int64_t cum_tok = 0, cum_blk = 0;
    for (int i : in.waiting) {
      const int64_t t = r[i].eff, b = blk(r[i].eff);
      if (adm.empty()) {
        if (b > in.kv_free) break;  // first request: block check only (G27)
      } else if (!(cum_tok + t <= limit && cum_blk + b <= in.kv_free)) {
        break;
      }
      adm.push_back(i);
      cum_tok += t;
      cum_blk += b;
    }
    for (int i : adm) admit(in, k, i, T);
    return !adm.empty();
  }

  void form_hp(int k, int64_t T) {
    Inst& in = I[k];
    std::vector<int> dropped = drop_step(in, T);
    evaluations += (int64_t)in.waiting.size();
    std::vector<int> adm, pre;
    int64_t l = 0, bd = 0;
    bool batch = false;
    if (!in.waiting.empty()) batch = hp_prefill(in, k, T, adm);  // prefill first
    if (!batch && !in.D.empty()) {
      pre = decode_prep(in);
      if (!in.D.empty()) { batch = true; bd = (int64_t)in.D.size(); }
      else if (!in.waiting.empty()) batch = hp_prefill(in, k, T, adm);  // all decodes evicted
    }
    if (batch) {
      l = bd ? lat({}, in.D) : lat(adm, {});
      in.busy = true;
      in.end = T + l;
      in.batch_pf = adm;
      in.batch_dec = bd > 0;
      decisions++;
    }
    if (batch || !dropped.empty() || !pre.empty())
      log(in, T, k, adm, bd, {}, dropped, pre, l);
  }

  // vLLM-like baseline ("prefill-prioritizing"; reading G46): every instance is
  // homogeneous; at each formation the waiting queue is ordered by the policy key (FCFS = arrival:
  // vLLM) and, if any request fits, a prefill-only batch of the longest prefix with
  // sum(tokens) <= N, sum(blocks) <= free blocks and |D| + count <= batch cap is run while the
  // decodes stall; otherwise every decode runs (decode-only), after preemption by recomputation
  // if their growth does not fit.
  std::vector<int> vllm_prefill(Inst& in, int k, int64_t T) {
    std::sort(in.waiting.begin(), in.waiting.end(), [&](int x, int y) {
      const int64_t kx = key(x), ky = key(y);
      return kx != ky ? kx < ky : x < y;
    });
    std::vector<int> adm;
    int64_t tok = 0, blocks = 0;
    for (int i : in.waiting) {
      const int64_t t = r[i].eff, b = blk(r[i].eff);
      if (tok + t > sc->lp_tok || blocks + b > in.kv_free ||
          (int64_t)in.D.size() + (int64_t)adm.size() + 1 > sc->lp_max_batch)
        break;
      adm.push_back(i);
      tok += t;
      blocks += b;
    }
    for (int i : adm) admit(in, k, i, T);
    return adm;
  }

  void form_vllm(int k, int64_t T) {
    Inst& in = I[k];
    std::vector<int> dropped = drop_step(in, T);
    evaluations += (int64_t)in.waiting.size();
    std::vector<int> adm, pre;
    int64_t l = 0, bd = 0;
    if (!in.waiting.empty()) adm = vllm_prefill(in, k, T);  // prefill first: decodes stall
    if (adm.empty() && !in.D.empty()) {
      pre = decode_prep(in);
      if (!in.D.empty()) bd = (int64_t)in.D.size();
      else if (!in.waiting.empty()) adm = vllm_prefill(in, k, T);  // every decode was evicted
    }
    const bool batch = !adm.empty() || bd > 0;
    if (batch) {
      l = bd ? lat({}, in.D) : lat(adm, {});
      in.busy = true;
      in.end = T + l;
      in.batch_pf = adm;
      in.batch_dec = bd > 0;
      decisions++;
    }
    if (batch || !dropped.empty() || !pre.empty())
      log(in, T, k, adm, bd, {}, dropped, pre, l);
  }

  // Sarathi-like baseline ("chunked prefill, allowing a partial prefill request to be
  // appended at the end of each decoding batch"; reading G47).  Each formation: drop
  // step; decode preparation (growth, LIFO preemption); then every decode runs and the rest of
  // the per-batch token budget (chunk_tokens - |D|) is filled in queue order — a partially
  // prefilled request first, then by (key, id) — each request contributing
  // c = min(budget left, prompt left), stopping at the first request whose blocks (prompt tokens
  // prefilled so far, + 1 for the first output token on the last chunk) do not fit, or at the
  // batch cap.  Chunked requests stay in the queue until their last chunk completes.
  void form_sarathi(int k, int64_t T) {
    Inst& in = I[k];
    std::vector<int> dropped = drop_step(in, T);
    std::vector<int> pre = decode_prep(in);
    evaluations += (int64_t)in.waiting.size();
    std::sort(in.waiting.begin(), in.waiting.end(), [&](int x, int y) {
      const bool px = r[x].cdone > 0, py = r[y].cdone > 0;
      if (px != py) return px;
      const int64_t kx = key(x), ky = key(y);
      return kx != ky ? kx < ky : x < y;
    });
    int64_t budget = (int64_t)sc->chunk_tokens - (int64_t)in.D.size();
    int64_t kv = in.kv_free;
    std::vector<int> ids;
    std::vector<int64_t> ls, cs;
    for (int i : in.waiting) {
      if (budget <= 0 || (int64_t)in.D.size() + (int64_t)ids.size() + 1 > sc->lp_max_batch) break;
      const int64_t rem = r[i].eff - r[i].cdone;
      const int64_t c = std::min(budget, rem);
      const int64_t target = c == rem ? blk(r[i].eff) : ceil_div(r[i].cdone + c, sc->bs);
      const int64_t need = target - r[i].held;
      if (need > kv) break;
      ids.push_back(i);
      ls.push_back(r[i].cdone);
      cs.push_back(c);
      budget -= c;
      kv -= need;
    }
    for (size_t j = 0; j < ids.size(); j++) {
      const int i = ids[j];
      const int64_t c = cs[j], rem = r[i].eff - r[i].cdone;
      const int64_t target = c == rem ? blk(r[i].eff) : ceil_div(r[i].cdone + c, sc->bs);
      r[i].ever = true;
      if (r[i].pstart < 0) r[i].pstart = T;
      r[i].inst = k;
      in.kv_free -= target - r[i].held;
      r[i].held = target;
      r[i].cdone += c;
    }
    const bool batch = !ids.empty() || !in.D.empty();
    int64_t l = 0;
    if (batch) {
      std::vector<int64_t> lh;
      for (int j : in.D) lh.push_back(r[j].p + r[j].g);
      uint64_t F, M;
      if (or_cost_chunked(a, (int32_t)ids.size(), ls.data(), cs.data(), (int32_t)lh.size(),
                          lh.data(), &F, &M)) {
        if (err.empty()) err = "range: batch cost reaches 2^53";
        l = -1;
      } else {
        l = or_latency_us(pf, F, M);
      }
      in.busy = true;
      in.end = T + l;
      in.batch_pf = ids;
      in.batch_dec = !in.D.empty();
      decisions++;
    }
    if (batch || !dropped.empty() || !pre.empty())
      log(in, T, k, ids, batch ? (int64_t)in.D.size() : 0, {}, dropped, pre, l, cs);
  }

  void log(Inst& in, int64_t T, int k, const std::vector<int>& adm, int64_t bd,
           const std::vector<int>& off, const std::vector<int>& dropped,
           const std::vector<int>& pre, int64_t l,
           const std::vector<int64_t>& chunks = {}) {
    std::vector<uint64_t> v;
    v.push_back((uint64_t)T);
    v.push_back((uint64_t)k);
    v.push_back((uint64_t)adm.size());
    for (int i : adm) v.push_back((uint64_t)i);
    v.push_back((uint64_t)bd);
    v.push_back((uint64_t)off.size());
    for (int i : off) v.push_back((uint64_t)i);
    v.push_back((uint64_t)dropped.size());
    for (int i : dropped) v.push_back((uint64_t)i);
    v.push_back((uint64_t)pre.size());
    for (int i : pre) v.push_back((uint64_t)i);
    v.push_back((uint64_t)l);
    for (int64_t c : chunks) v.push_back((uint64_t)c);  // Sarathi-like: chunk sizes, in order
    record(in, v);
  }

  bool invariants(int64_t T) {
    for (auto& in : I) {
      int64_t held = 0;
      for (int j : in.D) held += r[j].held;
      for (int i : in.batch_pf)  // (a Sarathi chunk is also in the queue: counted there)
        if (std::find(in.waiting.begin(), in.waiting.end(), i) == in.waiting.end()) held += r[i].held;
      for (int i : in.waiting) held += r[i].held;
      if (held + in.kv_free != in.kv_total || in.kv_free < 0) {
        err = "invariant: KV ledger at T=" + std::to_string(T);
        return false;
      }
      if (!in.hp && (int64_t)in.D.size() > sc->lp_max_batch) {
        err = "invariant: LP decode set exceeds batch cap";
        return false;
      }
    }
    return true;
  }

  bool run() {
    const int n = (int)r.size();
    const int K = sc->n_lp + sc->n_hp;
    if (sc->offload && sc->n_hp >= 1) Whp = pf_us(sc->hp_tok);
    int next = 0;
    for (int h = sc->n_lp; h < K; h++) if (sc->tickets) I[h].ticket = true;  // issued at t=0
    // Ticket rule (G29): an HP with an empty waiting queue and no resident ticketed
    // request holds one outstanding ticket.
    while (true) {
      int64_t T = INF64;
      if (next < n) T = std::min(T, r[next].arrival);
      for (auto& in : I) if (in.busy) T = std::min(T, in.end);
      for (auto& f : inflight) T = std::min(T, f.t);
      if (T == INF64) {
        for (auto& in : I)
          if (!in.waiting.empty() || !in.D.empty()) { err = "invariant: stuck queue"; return false; }
        return err.empty();
      }
      // A. completions, instance index order
      for (int k = 0; k < K; k++) if (I[k].busy && I[k].end == T) complete(k, T);
      // B. offload deliveries (FIFO by dispatch order)
      std::vector<Flight> rest;
      for (auto& f : inflight) { if (f.t == T) hp_insert(I[f.hp], f.req); else rest.push_back(f); }
      inflight = rest;
      // C. arrivals, ascending id
      while (next < n && r[next].arrival == T) route(next++);
      // D. formations of idle instances, LPs before HPs
      for (int k = 0; k < K; k++) {
        if (I[k].busy) continue;
        if (sc->scheduler == 1) form_vllm(k, T);
        else if (sc->scheduler == 2) form_sarathi(k, T);
        else if (I[k].hp) form_hp(k, T);
        else form_lp(k, T);
        if (!err.empty()) return false;
      }
      // E. ticket issue (G29)
      if (sc->tickets)
        for (int h = sc->n_lp; h < K; h++)
          if (!I[h].ticket && I[h].waiting.empty() && I[h].tk_live == 0) I[h].ticket = true;
      if (check && !invariants(T)) return false;
    }
  }
};

}  // namespace

static int simulate_one(const or_arch* a, const or_perf* pf, const or_sched* sc, int64_t n,
                        const int64_t* arr, const int32_t* pl, const int32_t* ol, int64_t ttft,
                        int64_t tbt, const int64_t* req_ttft, const int64_t* koff,
                        int64_t* first, int64_t* done,
                        int64_t* pstart, uint32_t* status, uint64_t* digest, int64_t* decisions,
                        int64_t* evaluations, bool check, std::string& err) {
  Sim s;
  s.a = a; s.pf = pf; s.sc = sc; s.tbt = tbt; s.check = check;
  s.r.resize(n);
  for (int64_t i = 0; i < n; i++) {
    Req& q = s.r[i];
    q.arrival = arr[i];
    q.ttft = req_ttft ? req_ttft[i] : ttft;
    q.deadline = q.arrival + q.ttft;
    q.p = pl[i]; q.o = ol[i]; q.eff = q.p;
    q.koff = koff ? koff[i] : 0;
  }
  const int K = sc->n_lp + sc->n_hp;
  s.I.resize(K);
  for (int k = 0; k < K; k++) {
    s.I[k].hp = k >= sc->n_lp;
    s.I[k].kv_total = s.I[k].kv_free = s.I[k].hp ? sc->kv_hp : sc->kv_lp;
  }
  const bool ok = s.run();
  for (int64_t i = 0; i < n; i++) {
    const Req& q = s.r[i];
    first[i] = q.first; done[i] = q.done; pstart[i] = q.pstart;
    uint32_t st = (uint32_t)q.state | (q.offloaded ? 4u : 0u) | (q.ticketed ? 8u : 0u);
    st |= ((uint32_t)(q.inst & 255)) << 4;
    st |= ((uint32_t)std::min<int64_t>(q.npre, 65535)) << 12;
    status[i] = st;
  }
  uint64_t d = 0;
  for (int k = 0; k < K; k++) d = mix(d ^ s.I[k].hash);
  *digest = d;
  *decisions = s.decisions;
  *evaluations = s.evaluations;
  if (!ok) err = s.err;
  return ok ? 0 : 7;
}

extern "C" int or_simulate_batch(const or_arch* a_in, const or_perf* pf, const or_sched* sc,
                                 int32_t T, const int64_t* off, const int64_t* arr,
                                 const int32_t* pl, const int32_t* ol, const int64_t* ttft,
                                 const int64_t* tbt, const int64_t* req_ttft,
                                 const int32_t* tr_nlp, const int32_t* tr_nhp,
                                 const int64_t* req_koff, int64_t* first,
                                 int64_t* done, int64_t* pstart, uint32_t* status,
                                 uint64_t* digest, int64_t* decisions, int64_t* evaluations,
                                 int32_t nthreads, int32_t check) {
  if (!check_cfg(a_in, pf)) return 2;
  if (sc->n_lp < 1 || sc->n_hp < 0 || sc->bs < 1 || sc->kv_lp < 1 || (sc->n_hp && sc->kv_hp < 1) ||
      sc->lp_max_batch < 1 || sc->lp_tok < 1 || sc->hp_tok < 1) {
    set_err("sched: bad topology"); return 2;
  }
  if (sc->scheduler < 0 || sc->scheduler > 2) { set_err("sched: unknown scheduler"); return 2; }
  if (sc->policy < 0 || sc->policy > 5 || sc->offload_rule < 0 || sc->offload_rule > 1) {
    set_err("sched: unknown policy or offload rule"); return 2;
  }
  if (sc->scheduler == 2 && sc->chunk_tokens < 1) { set_err("sched: chunk_tokens < 1"); return 2; }
  for (int32_t t = 0; t < T; t++) {
    const int32_t nl = tr_nlp ? tr_nlp[t] : sc->n_lp, nh = tr_nhp ? tr_nhp[t] : sc->n_hp;
    if (nl < 1 || nh < 0 || nl + nh > sc->n_lp + sc->n_hp || (sc->scheduler != 0 && nh != 0)) {
      set_err("trace topology: need n_lp >= 1, n_hp >= 0, n_lp + n_hp <= the configured pool"
              " (and n_hp = 0 for baselines)");
      return 2;
    }
  }
  if (sc->scheduler != 0 && sc->n_hp != 0) { set_err("sched: baseline schedulers take n_hp = 0"); return 2; }
  or_arch a;
  apply_tp(a_in, &a);
  // Liveness validation: every effective prompt fits the LP token
  // budget strictly and every request's KV fits an instance.
  for (int32_t t = 0; t < T; t++)
    for (int64_t i = off[t]; i < off[t + 1]; i++) {
      if (pl[i] < 1 || ol[i] < 1) { set_err("request: prompt/output < 1"); return 2; }
      if ((int64_t)pl[i] + ol[i] > sc->lp_tok) { set_err("request: prompt+output > lp_token_budget"); return 2; }
      const int64_t kvmin = sc->n_hp ? std::min(sc->kv_lp, sc->kv_hp) : sc->kv_lp;
      if (ceil_div((int64_t)pl[i] + ol[i], sc->bs) >= kvmin) { set_err("request: KV exceeds instance"); return 2; }
      if (i > off[t] && arr[i] < arr[i - 1]) { set_err("trace: arrivals not sorted"); return 1; }
    }
  std::atomic<int32_t> next{0};
  std::atomic<int> rc{0};
  std::string first_err;
  std::mutex mu;
  auto worker = [&]() {
    while (true) {
      const int32_t t = next.fetch_add(1);
      if (t >= T) break;
      const int64_t lo = off[t], n = off[t + 1] - off[t];
      std::string e;
      or_sched sct = *sc;  // the trace's subgroup topology (row f3)
      if (tr_nlp) sct.n_lp = tr_nlp[t];
      if (tr_nhp) sct.n_hp = tr_nhp[t];
      const int st = simulate_one(&a, pf, &sct, n, arr + lo, pl + lo, ol + lo, ttft[t], tbt[t],
                                  req_ttft ? req_ttft + lo : nullptr,
                                  req_koff ? req_koff + lo : nullptr, first + lo, done + lo,
                                  pstart + lo, status + lo, digest + t, decisions + t,
                                  evaluations + t, check != 0, e);
      if (st) {
        std::lock_guard<std::mutex> lk(mu);
        if (rc.load() == 0) { rc.store(st); first_err = e; }
      }
    }
  };
  int nt = nthreads > 0 ? nthreads : (int)std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  if (nt > T) nt = T > 0 ? T : 1;
  std::vector<std::thread> th;
  for (int i = 1; i < nt; i++) th.emplace_back(worker);
  worker();
  for (auto& x : th) x.join();
  if (rc.load()) set_err(first_err);
  return rc.load();
}

// Goodput (G35-G36): a request counts iff it completed, its TTFT met the SLO
// and its mean TBT (done - first) / (out - 1) met the TBT SLO; dropped/unfinished count in total.
extern "C" int or_goodput(int32_t T, const int64_t* off, const int64_t* arr, const int32_t* ol,
                          const int64_t* ttft, const int64_t* tbt, const int64_t* req_ttft,
                          const int64_t* first, const int64_t* done, const uint32_t* status,
                          uint64_t* good, uint64_t* total) {
  int rc = 0;
  for (int32_t t = 0; t < T; t++) {
    uint64_t g = 0;
    for (int64_t i = off[t]; i < off[t + 1]; i++) {
      if ((status[i] & 3u) != COMPLETED) continue;
      const int64_t slo = req_ttft ? req_ttft[i] : ttft[t];
      if (first[i] - arr[i] > slo) continue;
      if (ol[i] > 1 && done[i] - first[i] > tbt[t] * (int64_t)(ol[i] - 1)) continue;
      g++;
    }
    good[t] = g;
    total[t] = (uint64_t)(off[t + 1] - off[t]);
    if (total[t] == 0) { rc = 5; set_err("goodput: empty trace"); }
  }
  return rc;
}

// Outcome summary (row a8; "(a) P99 TTFT, (b) Mean TBT, (c) System throughput, and (d)
// Request scheduling delay"; G52).  Plain loops per trace; the percentiles sort
// the trace's TTFTs and take the nearest-rank order statistic.
static int64_t nearest_rank(const std::vector<int64_t>& sorted, int64_t q) {
  const int64_t n = (int64_t)sorted.size();
  if (n == 0) return -1;
  int64_t k = (q * n + 99) / 100;  // ceil(q n / 100)
  if (k < 1) k = 1;
  return sorted[(size_t)(k - 1)];
}

extern "C" int or_summarize(int32_t T, const int64_t* off, const int64_t* arr, const int32_t* ol,
                            const int64_t* ttft, const int64_t* tbt, const int64_t* req_ttft,
                            const int32_t* trace_n_lp, int32_t n_lp, const int64_t* first,
                            const int64_t* done, const int64_t* pstart, const uint32_t* status,
                            int64_t* completed, int64_t* dropped, int64_t* violating,
                            int64_t* tokens, int64_t* p50, int64_t* p90, int64_t* p99,
                            int64_t* tbt_sum, int64_t* tbt_tok, int64_t* dsum_lp, int64_t* dcnt_lp,
                            int64_t* dsum_hp, int64_t* dcnt_hp, int64_t* last_done) {
  for (int32_t t = 0; t < T; t++) {
    const int32_t nl = trace_n_lp ? trace_n_lp[t] : n_lp;
    int64_t c = 0, d = 0, v = 0, tok = 0, ts = 0, tt = 0, sl = 0, cl = 0, sh = 0, ch = 0, ld = -1;
    std::vector<int64_t> ttfts;
    for (int64_t i = off[t]; i < off[t + 1]; i++) {
      const uint32_t state = status[i] & 3u;
      if (first[i] >= 0) ttfts.push_back(first[i] - arr[i]);
      if (pstart[i] >= 0) {
        const int32_t inst = (int32_t)((status[i] >> 4) & 255u);
        if (inst < nl) { sl += pstart[i] - arr[i]; cl++; }
        else { sh += pstart[i] - arr[i]; ch++; }
      }
      if (state == DROPPED) d++;
      if (state != COMPLETED) continue;
      c++;
      tok += ol[i];
      if (done[i] > ld) ld = done[i];
      if (ol[i] > 1) { ts += done[i] - first[i]; tt += ol[i] - 1; }
      const int64_t slo = req_ttft ? req_ttft[i] : ttft[t];
      const bool good = first[i] - arr[i] <= slo &&
                        (ol[i] == 1 || done[i] - first[i] <= tbt[t] * (int64_t)(ol[i] - 1));
      if (!good) v++;
    }
    std::sort(ttfts.begin(), ttfts.end());
    if (completed) completed[t] = c;
    if (dropped) dropped[t] = d;
    if (violating) violating[t] = v;
    if (tokens) tokens[t] = tok;
    if (p50) p50[t] = nearest_rank(ttfts, 50);
    if (p90) p90[t] = nearest_rank(ttfts, 90);
    if (p99) p99[t] = nearest_rank(ttfts, 99);
    if (tbt_sum) tbt_sum[t] = ts;
    if (tbt_tok) tbt_tok[t] = tt;
    if (dsum_lp) dsum_lp[t] = sl;
    if (dcnt_lp) dcnt_lp[t] = cl;
    if (dsum_hp) dsum_hp[t] = sh;
    if (dcnt_hp) dcnt_hp[t] = ch;
    if (last_done) last_done[t] = ld;
  }
  return 0;
}
