// summary.cu — row a8's outcome summary per trace (asc_summarize).
//
// PAPER P:579-584 (Fig. 10: "(a) P99 TTFT, (b) Mean TBT, (c) System throughput, and (d) Request
// scheduling delay of all instances"; "HP requests wait 4x less than LP requests")
// (goodput), SPEC S:543-590 (metrics module: nearest-rank percentiles S:567-573, counts, tokens,
// HP-path scheduling delay reported apart from the LP path S:583), reading G52.
//
// One CTA per trace.  Pass 0 streams the trace's outcomes once: counts, token and TBT sums, the
// LP/HP scheduling-delay split and the largest TTFT.  The three TTFT percentiles are then found
// together by an 11-bit radix select over the non-negative TTFT values (first_token - arrival of
// every request with a first token): each pass histograms, per wanted rank, the next digit of
// the values whose higher digits equal that rank's prefix so far, and a block scan of the
// histogram picks the digit holding the rank.  The number of passes follows from the largest
// TTFT (ceil(bits / 11), three at most for TTFTs below 2^33 us); each pass re-reads 16 B per
// request.  Integer results only, so they equal the oracle's sort-and-index exactly.
#include "asc_internal.h"

namespace {

constexpr int SB = 256;                 // threads per CTA
constexpr int NW = SB / 32;
constexpr int DIG = 11, NB = 1 << DIG;  // radix digit
constexpr int NQ = 3;                   // p50, p90, p99
constexpr int BPT = NB / SB;            // histogram bins per thread in the scan (8)
constexpr int NS = 11;                  // int64 sums of pass 0

struct SumPtrs {
  int64_t *completed, *dropped, *violating, *tokens, *p[NQ], *tbt_sum, *tbt_tok, *dsum_lp,
      *dcnt_lp, *dsum_hp, *dcnt_hp, *last_done;
};

__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
  #pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int64_t warp_max64(int64_t v) {
  #pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, (int64_t)__shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void __launch_bounds__(SB) summary_kernel(
    int32_t T, const int64_t* __restrict__ off, const int64_t* __restrict__ arr,
    const int32_t* __restrict__ ol, const int64_t* __restrict__ ttft, const int64_t* __restrict__ tbt,
    const int64_t* __restrict__ rttft, const int32_t* __restrict__ tr_nlp, int32_t n_lp,
    const int64_t* __restrict__ first, const int64_t* __restrict__ done,
    const int64_t* __restrict__ pstart, const uint32_t* __restrict__ status, SumPtrs o) {
  __shared__ uint32_t hist[NQ][NB];
  __shared__ int64_t red[NS + 2][NW];
  __shared__ int64_t tot[NS + 2];
  __shared__ uint32_t wscan[NQ][NW];
  __shared__ uint32_t sel_b[NQ], sel_k[NQ];
  const int t = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t lo = off[t], hi = off[t + 1];
  const int64_t slo_t = ttft[t], tb = tbt[t];
  const int32_t nl = tr_nlp ? tr_nlp[t] : n_lp;

  // ---- pass 0: counts, sums, the TTFT count and maximum, the latest completion ----------------
  int64_t s[NS] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  int64_t mx_ttft = 0, last = -1;
  #pragma unroll 1
  for (int64_t i = lo + tid; i < hi; i += SB) {
    const uint32_t st = __ldg(status + i);
    const int64_t a = __ldg(arr + i), f = __ldg(first + i), d = __ldg(done + i), ps = __ldg(pstart + i);
    const int32_t out = __ldg(ol + i);
    const int64_t slo = rttft ? __ldg(rttft + i) : slo_t;
    const uint32_t state = st & 3u;
    if (f >= 0) { s[10] += 1; mx_ttft = max(mx_ttft, f - a); }
    if (ps >= 0) {
      if ((int32_t)((st >> 4) & 255u) < nl) { s[6] += ps - a; s[7] += 1; }
      else { s[8] += ps - a; s[9] += 1; }
    }
    s[1] += state == 2u;
    if (state == 1u) {
      s[0] += 1;
      s[3] += out;
      last = max(last, d);
      if (out > 1) { s[4] += d - f; s[5] += out - 1; }
      const bool good = f - a <= slo && (out == 1 || d - f <= tb * (int64_t)(out - 1));
      s[2] += good ? 0 : 1;
    }
  }
  #pragma unroll
  for (int k = 0; k < NS; k++) {
    const int64_t v = warp_sum64(s[k]);
    if (lane == 0) red[k][wid] = v;
  }
  {
    const int64_t a = warp_max64(mx_ttft), b = warp_max64(last);
    if (lane == 0) { red[NS][wid] = a; red[NS + 1][wid] = b; }
  }
  __syncthreads();
  if (tid < NS + 2) {
    int64_t v = tid < NS ? 0 : (tid == NS ? 0 : -1);
    for (int w = 0; w < NW; w++) v = tid < NS ? v + red[tid][w] : max(v, red[tid][w]);
    tot[tid] = v;
  }
  __syncthreads();

  // ---- TTFT percentiles: radix select of the ranks ceil(q n / 100), q = 50, 90, 99 -------------
  const int64_t n = tot[10];
  uint64_t prefix[NQ] = {0, 0, 0};
  uint32_t kr[NQ];
  const int64_t qs[NQ] = {50, 90, 99};
  #pragma unroll
  for (int r = 0; r < NQ; r++) kr[r] = (uint32_t)max((int64_t)1, (qs[r] * n + 99) / 100);
  if (n > 0) {
    const uint64_t mx = (uint64_t)tot[NS];
    const int bits = mx ? 64 - __clzll((long long)mx) : 1;
    const int passes = (bits + DIG - 1) / DIG;
    #pragma unroll 1
    for (int p = 0; p < passes; p++) {
      const int shift = DIG * (passes - 1 - p);
      for (int j = tid; j < NQ * NB; j += SB) (&hist[0][0])[j] = 0u;
      __syncthreads();
      #pragma unroll 1
      for (int64_t i = lo + tid; i < hi; i += SB) {
        const int64_t f = __ldg(first + i);
        if (f < 0) continue;
        const uint64_t v = (uint64_t)(f - __ldg(arr + i));
        const uint32_t dg = (uint32_t)(v >> shift) & (NB - 1);
        const uint64_t up = p == 0 ? 0 : v >> (shift + DIG);
        #pragma unroll
        for (int r = 0; r < NQ; r++)
          if (up == prefix[r]) atomicAdd(&hist[r][dg], 1u);
      }
      __syncthreads();
      // block exclusive scan of the per-thread bin sums (BPT consecutive bins per thread)
      uint32_t ls[NQ];
      #pragma unroll
      for (int r = 0; r < NQ; r++) {
        uint32_t x = 0;
        #pragma unroll
        for (int j = 0; j < BPT; j++) x += hist[r][tid * BPT + j];
        ls[r] = x;
        uint32_t inc = x;
        #pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
          if (lane >= d) inc += y;
        }
        if (lane == 31) wscan[r][wid] = inc;
        ls[r] = inc - x;  // exclusive within the warp
      }
      __syncthreads();
      #pragma unroll
      for (int r = 0; r < NQ; r++) {
        uint32_t base = ls[r];
        for (int w = 0; w < wid; w++) base += wscan[r][w];
        uint32_t cum = base;
        #pragma unroll 1
        for (int j = 0; j < BPT; j++) {
          const uint32_t h = hist[r][tid * BPT + j];
          if (cum < kr[r] && kr[r] <= cum + h) { sel_b[r] = tid * BPT + j; sel_k[r] = kr[r] - cum; }
          cum += h;
        }
      }
      __syncthreads();
      #pragma unroll
      for (int r = 0; r < NQ; r++) {
        prefix[r] = (prefix[r] << DIG) | sel_b[r];
        kr[r] = sel_k[r];
      }
      __syncthreads();
    }
  }

  if (tid == 0) {
    if (o.completed) o.completed[t] = tot[0];
    if (o.dropped) o.dropped[t] = tot[1];
    if (o.violating) o.violating[t] = tot[2];
    if (o.tokens) o.tokens[t] = tot[3];
    if (o.tbt_sum) o.tbt_sum[t] = tot[4];
    if (o.tbt_tok) o.tbt_tok[t] = tot[5];
    if (o.dsum_lp) o.dsum_lp[t] = tot[6];
    if (o.dcnt_lp) o.dcnt_lp[t] = tot[7];
    if (o.dsum_hp) o.dsum_hp[t] = tot[8];
    if (o.dcnt_hp) o.dcnt_hp[t] = tot[9];
    if (o.last_done) o.last_done[t] = tot[NS + 1];
    #pragma unroll
    for (int r = 0; r < NQ; r++)
      if (o.p[r]) o.p[r][t] = n > 0 ? (int64_t)prefix[r] : -1;
  }
}

}  // namespace

namespace asc {

asc_status launch_summary(asc_ctx* c, const asc_traces* tr, const asc_outcomes* out, asc_summary* s) {
  const int32_t T = tr->T;
  c->last_kernel_launches = 0;
  if (T <= 0) return ASC_OK;
  SumPtrs p{s->completed, s->dropped, s->violating, s->tokens,
            {s->ttft_p50_us, s->ttft_p90_us, s->ttft_p99_us}, s->tbt_sum_us, s->tbt_tokens,
            s->delay_sum_lp_us, s->delay_cnt_lp, s->delay_sum_hp_us, s->delay_cnt_hp,
            s->last_done_us};
  cudaEventRecord(c->ev0, c->stream);
  summary_kernel<<<(unsigned)T, SB, 0, c->stream>>>(
      T, tr->trace_off, tr->arrival_us, tr->output_len, tr->ttft_slo_us, tr->tbt_slo_us,
      tr->req_ttft_slo_us, tr->n_lp, c->cfg.topo.n_lp, out->first_token_us, out->done_us,
      out->prefill_start_us, out->status, p);
  cudaEventRecord(c->ev1, c->stream);
  c->timed = true;
  c->last_kernel_launches = 1;
  return cuda_check(c, cudaGetLastError(), "summary launch");
}

}  // namespace asc
