// step.cu — asc_schedule_step: the stateless LP decision over S segments.
//
// Design:
//   plan   : per segment, #warp-tasks = max(1, ceil(Q_s / 2048)); exclusive scans give each
//            segment its first task and (for segments of > 1 task) its first candidate slot.
//   k1     : one warp per task streams its <= 2048 entries once (coalesced 8+4+1 B per entry),
//            evaluates a1 (prefill latency via the ctx's device table), the key (a2), the drop and
//            offload predicates (a5, as ballot bitmasks) and keeps the 128 smallest (key, pos)
//            in a register-resident bitonic list (a3).  Single-task segments are finished in
//            place: Algorithm 1 prefix scan (a4), batch latency (a6), admitted bits removed from
//            the offload mask, ballot/popc compaction of offload and drop indices (a5).
//   k2     : one CTA per multi-task segment merges the per-task lists (bitonic, warp shuffles
//            + shared-memory tree), runs Algorithm 1, clears admitted bits, scans task counts.
//   k3     : one warp per multi-task task expands its masks into id-ascending output indices.
// HBM traffic per entry: 13 B read (+4 B prefill_us if requested) + 4 B per output index;
// multi-task segments add 0.25 B/entry of mask traffic and 1.5 KB per task of candidates.
#include "asc_internal.h"

using namespace asc;

namespace {

constexpr int KPL = 4;  // K = 128 = ASC_MAX_BATCH
constexpr int ITERS = 64;
constexpr int CH = 32 * ITERS;  // entries per warp task
constexpr int UNR = 4;
constexpr int WARPS = 8;
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_TILE = SCAN_ITEMS * SCAN_THREADS;

struct StepP {
  Model md;
  const int64_t* pf_tab;
  int32_t pt, bs, policy, drop, offl;
  int64_t W, margin;
  int32_t S;
  const int64_t* seg_off;
  const int64_t* now;
  const int64_t* dl;
  const int32_t* eff;
  const uint8_t* fl;
  const int32_t* dcnt;
  const int64_t* dctx;
  const int64_t* tbt;
  const int32_t *bN, *bM, *bR;
  int32_t *admit_idx, *admit_cnt, *off_idx, *off_cnt, *drop_idx, *drop_cnt;
  int64_t* blat;
  int32_t* pfout;
  int64_t* task_off;   // [S+1]
  int64_t* mtask_off;  // [S+1]
  int64_t* scan_tmp;   // block totals
  KI* cand;
  uint32_t *moff, *mdrop;
  int32_t *coff, *cdrop;
  int* err;
};

__device__ __forceinline__ int64_t pf_of(const StepP& P, int32_t p) {
  if (p < P.pt) return __ldg(P.pf_tab + p);
  const int64_t v = prefill_lat(P.md, (uint64_t)p);
  if (v < 0) { atomicOr(P.err, ERR_RANGE); return INT32_MAX; }
  return v;
}

__device__ __forceinline__ int64_t key_of(int policy, int64_t dl, int64_t pf) {
  switch (policy) {
    case 0: return dl - pf;          // EDF_LAXITY
    case 1: return dl;               // EDF_DEADLINE
    case 2: return pf;               // SJF
    case 3: return -pf;              // LJF
    default: return 0;               // FCFS: position order (entries are in arrival order)
  }
}

// ---------------------------------------------------------------- planning (two scans) ------
__global__ void plan_counts(StepP P) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s > P.S) return;
  if (s == P.S) { P.task_off[s] = 0; P.mtask_off[s] = 0; return; }
  const int64_t len = P.seg_off[s + 1] - P.seg_off[s];
  if (len < 0) atomicOr(P.err, ERR_INVAL);
  const int64_t nt = len <= CH ? 1 : (len + CH - 1) / CH;
  P.task_off[s] = nt;
  P.mtask_off[s] = nt > 1 ? nt : 0;
}

// block-local exclusive scan of (a, b) over tiles of SCAN_TILE; tile totals to tmp
__global__ void scan_tiles(int64_t* a, int64_t* b, int64_t n, int64_t* tmp) {
  __shared__ int64_t sa[SCAN_THREADS / 32], sb[SCAN_THREADS / 32];
  const int64_t base = blockIdx.x * (int64_t)SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  int64_t va[SCAN_ITEMS], vb[SCAN_ITEMS], ta = 0, tb = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    va[i] = base + i < n ? a[base + i] : 0;
    vb[i] = base + i < n ? b[base + i] : 0;
    ta += va[i];
    tb += vb[i];
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  int64_t ia = warp_incl_scan(ta), ib = warp_incl_scan(tb);
  if (l == 31) { sa[w] = ia; sb[w] = ib; }
  __syncthreads();
  if (w == 0) {
    int64_t x = l < SCAN_THREADS / 32 ? sa[l] : 0, y = l < SCAN_THREADS / 32 ? sb[l] : 0;
    int64_t xi = warp_incl_scan(x), yi = warp_incl_scan(y);
    if (l < SCAN_THREADS / 32) { sa[l] = xi - x; sb[l] = yi - y; }
    if (l == 31) { tmp[2 * blockIdx.x] = xi; tmp[2 * blockIdx.x + 1] = yi; }
  }
  __syncthreads();
  int64_t ea = sa[w] + ia - ta, eb = sb[w] + ib - tb;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    if (base + i < n) { a[base + i] = ea; b[base + i] = eb; }
    ea += va[i];
    eb += vb[i];
  }
}

__global__ void scan_totals(int64_t* tmp, int64_t nt) {  // one warp, exclusive in place
  int64_t ca = 0, cb = 0;
  for (int64_t i0 = 0; i0 < nt; i0 += 32) {
    const int64_t i = i0 + threadIdx.x;
    int64_t x = i < nt ? tmp[2 * i] : 0, y = i < nt ? tmp[2 * i + 1] : 0;
    int64_t xi = warp_incl_scan(x), yi = warp_incl_scan(y);
    if (i < nt) { tmp[2 * i] = ca + xi - x; tmp[2 * i + 1] = cb + yi - y; }
    ca += __shfl_sync(FULL, xi, 31);
    cb += __shfl_sync(FULL, yi, 31);
  }
}

__global__ void scan_add(int64_t* a, int64_t* b, int64_t n, const int64_t* tmp) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t t = i / SCAN_TILE;
  a[i] += tmp[2 * t];
  b[i] += tmp[2 * t + 1];
}

__device__ __forceinline__ int64_t find_seg(const int64_t* task_off, int32_t S, int64_t task) {
  int64_t lo = 0, hi = S;  // largest s with task_off[s] <= task
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(task_off + mid) <= task) lo = mid; else hi = mid;
  }
  return lo;
}

// ----------------------------------------------------------- Algorithm 1 over a sorted list --
// a[] holds the <= 128 smallest live entries in (key, pos) order.  Writes admitted positions,
// the batch latency, and returns k; `adm[r]` tells each lane which of its elements were admitted.
__device__ int finalize_segment(const StepP& P, int64_t s, const KI (&a)[KPL], bool (&adm)[KPL]) {
  const int lane = lane_id();
  const int64_t lo = P.seg_off[s];
  const int64_t N = P.bN[s], M = P.bM[s];
  int64_t R = P.bR[s];
  if (R > ASC_MAX_BATCH) { atomicOr(P.err, ERR_RANGE); R = ASC_MAX_BATCH; }
  const int64_t Bd = P.dcnt[s], sl = P.dctx[s];
  int64_t C = INF64;
  if (Bd > 0) {
    const int64_t d = lat_us(P.md, 0, 0, 0, 0, (uint64_t)Bd, (uint64_t)sl);
    if (d < 0) atomicOr(P.err, ERR_RANGE);
    C = P.tbt[s] - d;
  }
  int32_t p[KPL];
  int64_t ct = 0, cb = 0, cc = 0;
  int k = 0;
  bool go = true;
#pragma unroll
  for (int r = 0; r < KPL; r++) {
    const bool valid = a[r].i != INF32;
    p[r] = valid ? __ldg(P.eff + a[r].i) : 0;
    const int64_t pf = valid ? pf_of(P, p[r]) : 0;
    const int64_t bl = valid ? (int64_t)((p[r] + P.bs) / P.bs) : 0;
    const int64_t St = ct + warp_incl_scan((int64_t)p[r]);
    const int64_t Sb = cb + warp_incl_scan(bl);
    const int64_t Sc = cc + warp_incl_scan(pf);
    const int pos = r * 32 + lane;
    const bool ok = go && valid && St < N && Sb < M && Sc < C && pos < R;
    const uint32_t m = __ballot_sync(FULL, ok);
    const int cnt = (m == FULL) ? 32 : (__ffs(~m) - 1);
    adm[r] = go && lane < cnt;
    k += go ? cnt : 0;
    if (cnt < 32) go = false;
    ct = __shfl_sync(FULL, St, 31);
    cb = __shfl_sync(FULL, Sb, 31);
    cc = __shfl_sync(FULL, Sc, 31);
  }
  uint64_t sp = 0, sp2 = 0, spc = 0;
#pragma unroll
  for (int r = 0; r < KPL; r++) {
    if (adm[r]) {
      const uint64_t q = (uint64_t)p[r];
      sp += q;
      sp2 += q * q;
      spc += q * ceil_div_u(q, P.md.b);
      P.admit_idx[lo + r * 32 + lane] = a[r].i;
    }
  }
  sp = warp_sum(sp);
  sp2 = warp_sum(sp2);
  spc = warp_sum(spc);
  if (lane == 0) {
    P.admit_cnt[s] = k;
    int64_t l = 0;
    if (k > 0 || Bd > 0) {
      l = lat_us(P.md, (uint64_t)k, sp, sp2, spc, (uint64_t)Bd, (uint64_t)sl);
      if (l < 0) atomicOr(P.err, ERR_RANGE);
    }
    P.blat[s] = l;
  }
  return k;
}

// expand ballot words into output indices (id-ascending), starting at out + base
__device__ __forceinline__ int64_t expand_words(const uint32_t* words, int nw, int64_t first_e,
                                                int32_t* out, int64_t base) {
  const int lane = lane_id();
  for (int w = 0; w < nw; w++) {
    const uint32_t m = words[w];
    if (m == 0) continue;
    if ((m >> lane) & 1u) out[base + __popc(m & lanemask_lt())] = (int32_t)(first_e + w * 32 + lane);
    base += __popc(m);
  }
  return base;
}

__global__ void __launch_bounds__(WARPS * 32) k1_tasks(StepP P) {
  __shared__ KI sbuf[WARPS][64];
  __shared__ uint32_t s_off[WARPS][ITERS], s_drop[WARPS][ITERS];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntasks = P.task_off[P.S];
  for (int64_t task = blockIdx.x * (int64_t)WARPS + w; task < ntasks;
       task += (int64_t)gridDim.x * WARPS) {
    const int64_t s = find_seg(P.task_off, P.S, task);
    const int64_t c = task - P.task_off[s];
    const int64_t nt = P.task_off[s + 1] - P.task_off[s];
    const int64_t lo = P.seg_off[s], hi = P.seg_off[s + 1];
    const int64_t b = lo + c * CH;
    const int64_t e_end = min(hi, b + CH);
    const int64_t now = P.now[s];
    TopKStream<KPL> st;
    st.init(sbuf[w]);
    int nw = 0;
    for (int j0 = 0; j0 < ITERS && b + j0 * 32 < e_end; j0 += UNR) {
      int64_t dl[UNR];
      int32_t p[UNR];
      uint32_t f[UNR];
#pragma unroll
      for (int u = 0; u < UNR; u++) {
        const int64_t e = b + (j0 + u) * 32 + lane;
        if (e < e_end) {
          dl[u] = __ldcs(P.dl + e);
          p[u] = __ldcs(P.eff + e);
          f[u] = __ldcs(P.fl + e);
        } else {
          dl[u] = 0; p[u] = 1; f[u] = 0;
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; u++) {
        const int64_t e = b + (j0 + u) * 32 + lane;
        const bool v = e < e_end;
        if (v && p[u] < 1) atomicOr(P.err, ERR_INVAL);
        const int64_t pf = v ? pf_of(P, p[u] < 1 ? 1 : p[u]) : 0;
        if (v && P.pfout) {
          if (pf > INT32_MAX) atomicOr(P.err, ERR_RANGE);
          __stcs(P.pfout + e, (int32_t)pf);
        }
        const bool dropped = v && P.drop && !(f[u] & 1u) && now > dl[u];
        const bool off = v && P.offl && !dropped && !(f[u] & 3u) &&
                         dl[u] - now <= pf + P.W + P.margin;
        const uint32_t md = __ballot_sync(FULL, dropped), mo = __ballot_sync(FULL, off);
        if (lane == 0) { s_drop[w][j0 + u] = md; s_off[w][j0 + u] = mo; }
        st.push(KI{key_of(P.policy, dl[u], pf), (int32_t)e}, v && !dropped);
      }
      nw = j0 + UNR;
    }
    st.finish();
    __syncwarp();
    if (nt == 1) {
      bool adm[KPL];
      finalize_segment(P, s, st.top.a, adm);
      // an admitted request is not offloaded (only unscheduled requests)
#pragma unroll
      for (int r = 0; r < KPL; r++) {
        if (adm[r]) {
          const int64_t loc = st.top.a[r].i - b;
          atomicAnd(&s_off[w][loc >> 5], ~(1u << (loc & 31)));
        }
      }
      __syncwarp();
      const int64_t no = expand_words(s_off[w], nw, b, P.off_idx, lo);
      const int64_t nd = expand_words(s_drop[w], nw, b, P.drop_idx, lo);
      if (lane == 0) { P.off_cnt[s] = (int32_t)(no - lo); P.drop_cnt[s] = (int32_t)(nd - lo); }
    } else {
      const int64_t mt = P.mtask_off[s] + c;
      KI* cd = P.cand + mt * (32 * KPL);
#pragma unroll
      for (int r = 0; r < KPL; r++) cd[r * 32 + lane] = st.top.a[r];
      int32_t co = 0, cdp = 0;
      for (int j = lane; j < ITERS; j += 32) {
        const uint32_t mo = j < nw ? s_off[w][j] : 0u, mdp = j < nw ? s_drop[w][j] : 0u;
        P.moff[mt * ITERS + j] = mo;
        P.mdrop[mt * ITERS + j] = mdp;
        co += __popc(mo);
        cdp += __popc(mdp);
      }
      co = warp_sum(co);
      cdp = warp_sum(cdp);
      if (lane == 0) { P.coff[mt] = co; P.cdrop[mt] = cdp; }
    }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(WARPS * 32) k2_segments(StepP P) {
  __shared__ KI lists[WARPS][32 * KPL];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t s = blockIdx.x; s < P.S; s += gridDim.x) {
    const int64_t nt = P.task_off[s + 1] - P.task_off[s];
    if (nt <= 1) continue;
    const int64_t m0 = P.mtask_off[s];
    const int64_t lo = P.seg_off[s];
    WarpTopK<KPL> A;
    A.init();
    for (int64_t t = w; t < nt; t += WARPS) {
      KI B[KPL];
      const KI* cd = P.cand + (m0 + t) * (32 * KPL);
#pragma unroll
      for (int r = 0; r < KPL; r++) B[r] = cd[r * 32 + lane];
      A.merge_list(B);
    }
    for (int step = 1; step < WARPS; step <<= 1) {
      if ((w % (2 * step)) == step) {
#pragma unroll
        for (int r = 0; r < KPL; r++) lists[w][r * 32 + lane] = A.a[r];
      }
      __syncthreads();
      if ((w % (2 * step)) == 0 && w + step < WARPS) {
        KI B[KPL];
#pragma unroll
        for (int r = 0; r < KPL; r++) B[r] = lists[w + step][r * 32 + lane];
        A.merge_list(B);
      }
      __syncthreads();
    }
    if (w == 0) {
      bool adm[KPL];
      finalize_segment(P, s, A.a, adm);
#pragma unroll
      for (int r = 0; r < KPL; r++) {
        if (adm[r]) {
          const int64_t loc = A.a[r].i - lo;
          const int64_t t = loc / CH, j = (loc % CH) >> 5;
          const uint32_t bit = 1u << (loc & 31);
          const uint32_t old = atomicAnd(&P.moff[(m0 + t) * ITERS + j], ~bit);
          if (old & bit) atomicSub(&P.coff[m0 + t], 1);
        }
      }
    }
    __syncthreads();
    if (w == 0) {  // exclusive scan of per-task counts -> output offsets
      int64_t ca = 0, cb = 0;
      for (int64_t t0 = 0; t0 < nt; t0 += 32) {
        const int64_t t = t0 + lane;
        const int64_t x = t < nt ? P.coff[m0 + t] : 0, y = t < nt ? P.cdrop[m0 + t] : 0;
        const int64_t xi = warp_incl_scan(x), yi = warp_incl_scan(y);
        if (t < nt) { P.coff[m0 + t] = (int32_t)(ca + xi - x); P.cdrop[m0 + t] = (int32_t)(cb + yi - y); }
        ca += __shfl_sync(FULL, xi, 31);
        cb += __shfl_sync(FULL, yi, 31);
      }
      if (lane == 0) { P.off_cnt[s] = (int32_t)ca; P.drop_cnt[s] = (int32_t)cb; }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(WARPS * 32) k3_expand(StepP P) {
  const int w = threadIdx.x >> 5;
  const int64_t ntasks = P.task_off[P.S];
  for (int64_t task = blockIdx.x * (int64_t)WARPS + w; task < ntasks;
       task += (int64_t)gridDim.x * WARPS) {
    const int64_t s = find_seg(P.task_off, P.S, task);
    const int64_t nt = P.task_off[s + 1] - P.task_off[s];
    if (nt <= 1) continue;
    const int64_t c = task - P.task_off[s];
    const int64_t mt = P.mtask_off[s] + c;
    const int64_t lo = P.seg_off[s];
    const int64_t b = lo + c * CH;
    expand_words(P.moff + mt * ITERS, ITERS, b, P.off_idx, lo + P.coff[mt]);
    expand_words(P.mdrop + mt * ITERS, ITERS, b, P.drop_idx, lo + P.cdrop[mt]);
  }
}

}  // namespace

namespace asc {

asc_status launch_schedule_step(asc_ctx* c, const asc_step_in* in, asc_step_out* out, int64_t Q) {
  const int32_t S = in->S;
  const int64_t max_mt = 2 * (Q / CH) + 2;
  const int64_t ntile = (S + 1 + SCAN_TILE - 1) / SCAN_TILE;
  size_t need = 0;
  need += 2 * (size_t)(S + 1) * 8 + 2 * (size_t)ntile * 8 + 4096;
  need += (size_t)max_mt * (32 * KPL) * sizeof(KI) + (size_t)max_mt * ITERS * 8 + (size_t)max_mt * 8 + 8192;
  asc_status st = ensure_ws(c, need);
  if (st) return st;
  Arena ar{c->ws, c->ws_cap};
  StepP P;
  P.md = c->md;
  P.pf_tab = c->d_pf_tab;
  P.pt = c->pt_size;
  P.bs = c->cfg.topo.block_tokens;
  P.policy = c->cfg.flags.policy;
  P.drop = c->cfg.flags.drop;
  P.offl = (c->cfg.flags.offload && c->cfg.topo.n_hp >= 1) ? 1 : 0;
  P.W = c->w_hp;
  P.margin = c->cfg.flags.offload_margin_us;
  P.S = S;
  P.seg_off = in->seg_off; P.now = in->now_us; P.dl = in->deadline_us; P.eff = in->eff_prompt;
  P.fl = in->flags; P.dcnt = in->dec_count; P.dctx = in->dec_ctx_sum; P.tbt = in->tbt_slo_us;
  P.bN = in->budget_tokens; P.bM = in->budget_blocks; P.bR = in->budget_reqs;
  P.admit_idx = out->admit_idx; P.admit_cnt = out->admit_cnt; P.off_idx = out->offload_idx;
  P.off_cnt = out->offload_cnt; P.drop_idx = out->drop_idx; P.drop_cnt = out->drop_cnt;
  P.blat = out->batch_lat_us; P.pfout = out->prefill_us;
  P.task_off = ar.take<int64_t>(S + 1);
  P.mtask_off = ar.take<int64_t>(S + 1);
  P.scan_tmp = ar.take<int64_t>(2 * ntile);
  P.cand = ar.take<KI>(max_mt * 32 * KPL);
  P.moff = ar.take<uint32_t>(max_mt * ITERS);
  P.mdrop = ar.take<uint32_t>(max_mt * ITERS);
  P.coff = ar.take<int32_t>(max_mt);
  P.cdrop = ar.take<int32_t>(max_mt);
  P.err = c->d_err;
  cudaStream_t sm = c->stream;
  int64_t launches = 0;
  plan_counts<<<(S + 1 + 255) / 256, 256, 0, sm>>>(P);
  scan_tiles<<<ntile, SCAN_THREADS, 0, sm>>>(P.task_off, P.mtask_off, S + 1, P.scan_tmp);
  scan_totals<<<1, 32, 0, sm>>>(P.scan_tmp, ntile);
  scan_add<<<(S + 1 + 255) / 256, 256, 0, sm>>>(P.task_off, P.mtask_off, S + 1, P.scan_tmp);
  launches += 4;
  int dev_sms = 148;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c->device);
  const int64_t ntask_max = (int64_t)S + Q / CH + 1;
  int64_t g1 = (ntask_max + WARPS - 1) / WARPS;
  g1 = g1 < (int64_t)dev_sms * 8 ? g1 : (int64_t)dev_sms * 8;
  cudaEventRecord(c->ev0, sm);
  k1_tasks<<<(unsigned)(g1 > 0 ? g1 : 1), WARPS * 32, 0, sm>>>(P);
  cudaEventRecord(c->ev1, sm);
  c->timed = true;
  launches += 1;
  if (Q > CH) {
    int64_t g2 = S < (int64_t)dev_sms * 4 ? S : (int64_t)dev_sms * 4;
    k2_segments<<<(unsigned)(g2 > 0 ? g2 : 1), WARPS * 32, 0, sm>>>(P);
    k3_expand<<<(unsigned)(g1 > 0 ? g1 : 1), WARPS * 32, 0, sm>>>(P);
    launches += 2;
  }
  c->last_kernel_launches = launches;
  return cuda_check(c, cudaGetLastError(), "schedule_step launch");
}

}  // namespace asc
