// sim.cu — asc_simulate_batch: the batched discrete-event step loop (with
// rows a1-a6 inlined per formation) and asc_goodput (row a8).
//
// One warp owns one trace at a time (traces are handed out by an atomic counter so long traces
// do not serialise a static partition).  All per-trace state stays resident in HBM/L2:
//   per request  : deadline (int64), effective prompt (int32), flag word (uint32)
//   per instance : waiting queue (id, key) with time-invariant keys, decode set
//                  slots (id, context l̂, blocks held, tokens remaining), running-batch prefill list
//   per trace    : drop / preemption / offload scratch lists and the in-flight offload ring
// Instance scalars (busy, end, kv_free, ticket, history, digest) live in shared memory.  Every
// queue operation is warp-parallel: ballot/popc stable compaction, warp scans, the bitonic top-K
// of asc_dev.cuh for Algorithm 1's sort, warp reductions for the batch moments of Eq. 1-3.
// The event order is the canonical A-E phase order of DESIGN.md §Event loop.
#include "asc_internal.h"

using namespace asc;

namespace {

constexpr int KPL = 4;
constexpr int SW = 4;  // warps (traces in flight) per CTA
constexpr int MAXI = ASC_MAX_INSTANCES;

enum : uint32_t { F_EVER = 1u, F_ONHP = 2u, F_TICK = 4u, F_OFFL = 8u };
constexpr uint32_t ST_SHIFT = 4, INST_SHIFT = 8, NPRE_SHIFT = 16;

struct SInst {
  int64_t end, hist_sum;
  uint64_t hash;
  int32_t kv_free, kv_total, wq_len, ds_len, bp_len, hist_cnt;
  int32_t busy, batch_dec, ticket, tk_live, hp, pad;
};

struct SimP {
  Model md;
  const int64_t* pf_tab;
  int32_t pt;
  int32_t n_lp, n_hp, K, bs, lp_max, lp_tok, hp_tok, policy, offl, tickets, elastic, drop, hist_def;
  int32_t kv_lp, kv_hp;
  int64_t W, margin, delay;
  int32_t T;
  const int64_t* off;
  const int64_t* arr;
  const int32_t* pl;
  const int32_t* ol;
  const int64_t* ttft;
  const int64_t* tbt;
  const int64_t* rttft;
  int64_t *first, *done, *pstart;
  uint32_t* status;
  uint64_t* digest;
  int64_t *decisions, *evals;
  int64_t R;
  int64_t* rq_dl;
  int32_t* rq_eff;
  uint32_t* rq_fl;
  int64_t* wq_key;
  int32_t* wq_id;
  int32_t *ds_id, *ds_ctx, *ds_held, *ds_rem;
  int32_t* bp_id;
  int32_t *scr_drop, *scr_pre, *scr_off;
  int64_t* fl_t;
  int32_t *fl_req, *fl_hp;
  int* err;
  int* next_trace;
};

struct Tr {  // per-trace registers (uniform across the warp)
  int64_t base, n, tbt;
  int64_t next, fl_head, fl_tail, decisions, evals;
  int32_t rr_lp, rr_hp;
};

__device__ __forceinline__ int64_t pf_of(const SimP& P, int32_t p) {
  if (p < P.pt) return __ldg(P.pf_tab + p);
  const int64_t v = prefill_lat(P.md, (uint64_t)p);
  if (v < 0) { atomicOr(P.err, ERR_RANGE); return INT32_MAX; }
  return v;
}
__device__ __forceinline__ int32_t blk_of(const SimP& P, int32_t eff) { return (eff + P.bs) / P.bs; }

// time-invariant priority key of request gid with effective prompt eff
__device__ __forceinline__ int64_t key_of(const SimP& P, int64_t gid, int32_t eff) {
  switch (P.policy) {
    case 0: return P.rq_dl[gid] - pf_of(P, eff);
    case 1: return P.rq_dl[gid];
    case 2: return pf_of(P, eff);
    case 3: return -pf_of(P, eff);
    default: return P.arr[gid];
  }
}

__device__ __forceinline__ int64_t ioff(const SimP& P, int k, const Tr& t) { return (int64_t)k * P.R + t.base; }

// ---------------------------------------------------------------------------- queue helpers ---
__device__ void wq_append(const SimP& P, SInst& I, int k, const Tr& t, int32_t id) {
  const int64_t o = ioff(P, k, t);
  const int32_t len = I.wq_len;
  if (lane_id() == 0) {
    P.wq_id[o + len] = id;
    P.wq_key[o + len] = key_of(P, t.base + id, P.rq_eff[t.base + id]);
    I.wq_len = len + 1;
  }
  __syncwarp();
}

// HP waiting queues are kept in ascending id order = FCFS by (arrival, id) (G26)
__device__ void wq_insert_sorted(const SimP& P, SInst& I, int k, const Tr& t, int32_t id) {
  const int lane = lane_id();
  const int64_t o = ioff(P, k, t);
  const int32_t len = I.wq_len;
  int32_t pos = 0;
  for (int32_t c = 0; c < len; c += 32) {
    const int32_t j = c + lane;
    pos += __popc(__ballot_sync(FULL, j < len && P.wq_id[o + j] < id));
  }
  for (int32_t c = len - 1; c >= pos; c -= 32) {
    const int32_t j = c - lane;
    int32_t xi = 0;
    int64_t xk = 0;
    const bool v = j >= pos;
    if (v) { xi = P.wq_id[o + j]; xk = P.wq_key[o + j]; }
    __syncwarp();
    if (v) { P.wq_id[o + j + 1] = xi; P.wq_key[o + j + 1] = xk; }
    __syncwarp();
  }
  if (lane == 0) {
    P.wq_id[o + pos] = id;
    P.wq_key[o + pos] = key_of(P, t.base + id, P.rq_eff[t.base + id]);
    I.wq_len = len + 1;
  }
  __syncwarp();
}

__device__ __forceinline__ void set_state(const SimP& P, int64_t gid, uint32_t st) {
  uint32_t f = P.rq_fl[gid];
  P.rq_fl[gid] = (f & ~(3u << ST_SHIFT)) | (st << ST_SHIFT);
}

// Drop rule (G34): waiting, never prefilled, strictly past the deadline.  Stable
// compaction of the queue; dropped ids (queue order = ascending id) go to scr_drop.
__device__ int32_t drop_step(const SimP& P, SInst& I, int k, const Tr& t, int64_t T) {
  if (!P.drop || I.wq_len == 0) return 0;
  const int lane = lane_id();
  const int64_t o = ioff(P, k, t);
  const int32_t len = I.wq_len;
  int32_t out = 0, nd = 0, tkd = 0;
  for (int32_t c = 0; c < len; c += 32) {
    const int32_t j = c + lane;
    const bool v = j < len;
    int32_t id = 0;
    int64_t key = 0;
    bool dr = false;
    if (v) {
      id = P.wq_id[o + j];
      key = P.wq_key[o + j];
      const int64_t g = t.base + id;
      dr = !(P.rq_fl[g] & F_EVER) && T > P.rq_dl[g];
    }
    const uint32_t mk = __ballot_sync(FULL, v && !dr), md = __ballot_sync(FULL, dr);
    __syncwarp();
    if (v && !dr) { const int32_t q = out + __popc(mk & lanemask_lt()); P.wq_id[o + q] = id; P.wq_key[o + q] = key; }
    if (dr) {
      const int64_t g = t.base + id;
      P.scr_drop[t.base + nd + __popc(md & lanemask_lt())] = id;
      set_state(P, g, 2u);
      if (I.hp && (P.rq_fl[g] & F_TICK)) tkd++;
    }
    out += __popc(mk);
    nd += __popc(md);
    __syncwarp();
  }
  tkd = warp_sum(tkd);
  if (lane == 0) { I.wq_len = out; I.tk_live -= tkd; }
  __syncwarp();
  return nd;
}

// Decode preparation (§5.4): grow each decode's KV by the blocks its next token
// needs; while short of blocks, evict the latest-arrived decode (LIFO, G31) by recomputation:
// its generated tokens join its prompt and it re-enters this instance's queue.
__device__ int32_t decode_prep(const SimP& P, SInst& I, int k, const Tr& t) {
  const int lane = lane_id();
  const int64_t o = ioff(P, k, t);
  int32_t np = 0;
  while (true) {
    const int32_t len = I.ds_len;
    int64_t need = 0;
    int32_t best = -1, bslot = -1;
    for (int32_t c = 0; c < len; c += 32) {
      const int32_t j = c + lane;
      if (j < len) {
        const int32_t ctx = P.ds_ctx[o + j];
        need += (ctx + P.bs - 1) / P.bs - P.ds_held[o + j];
        const int32_t id = P.ds_id[o + j];
        if (id > best) { best = id; bslot = j; }
      }
    }
    need = warp_sum(need);
    if (need <= I.kv_free) break;
    const int32_t vid = warp_max(best);
    const uint32_t who = __ballot_sync(FULL, best == vid);
    const int32_t vslot = __shfl_sync(FULL, bslot, __ffs(who) - 1);
    const int32_t held = P.ds_held[o + vslot], ctx = P.ds_ctx[o + vslot];
    const int64_t g = t.base + vid;
    __syncwarp();
    if (lane == 0) {
      I.kv_free += held;
      P.rq_eff[g] = ctx;
      P.rq_fl[g] += (1u << NPRE_SHIFT);
      P.scr_pre[t.base + np] = vid;
      const int32_t last = len - 1;
      P.ds_id[o + vslot] = P.ds_id[o + last];
      P.ds_ctx[o + vslot] = P.ds_ctx[o + last];
      P.ds_held[o + vslot] = P.ds_held[o + last];
      P.ds_rem[o + vslot] = P.ds_rem[o + last];
      I.ds_len = last;
    }
    __syncwarp();
    np++;
    if (I.hp) wq_insert_sorted(P, I, k, t, vid); else wq_append(P, I, k, t, vid);
  }
  const int32_t len = I.ds_len;
  int64_t grow = 0;
  for (int32_t c = 0; c < len; c += 32) {
    const int32_t j = c + lane;
    if (j < len) {
      const int32_t need = (P.ds_ctx[o + j] + P.bs - 1) / P.bs;
      const int32_t gr = need - P.ds_held[o + j];
      if (gr) P.ds_held[o + j] = need;
      grow += gr;
    }
  }
  grow = warp_sum(grow);
  __syncwarp();
  if (lane == 0) I.kv_free -= (int32_t)grow;
  __syncwarp();
  return np;
}

__device__ __forceinline__ int64_t ds_ctx_sum(const SimP& P, const SInst& I, int k, const Tr& t) {
  const int64_t o = ioff(P, k, t);
  int64_t s = 0;
  for (int32_t j = lane_id(); j < I.ds_len; j += 32) s += P.ds_ctx[o + j];
  return warp_sum(s);
}

// mark request admitted at T on instance k
__device__ __forceinline__ void admit_req(const SimP& P, int64_t g, int k, int64_t T) {
  uint32_t f = P.rq_fl[g];
  f = (f & ~(0xffu << INST_SHIFT)) | ((uint32_t)k << INST_SHIFT) | F_EVER;
  P.rq_fl[g] = f;
  if (P.pstart[g] < 0) P.pstart[g] = T;
}

__device__ void digest_log(const SimP& P, SInst& I, int k, const Tr& t, int64_t T, int32_t nadm,
                           int64_t bd, int32_t noff, int32_t ndrop, int32_t npre, int64_t lat) {
  if (lane_id() == 0) {
    const int64_t o = ioff(P, k, t);
    uint64_t h = I.hash;
    h = mix64(h ^ (uint64_t)T);
    h = mix64(h ^ (uint64_t)k);
    h = mix64(h ^ (uint64_t)nadm);
    for (int32_t j = 0; j < nadm; j++) h = mix64(h ^ (uint64_t)P.bp_id[o + j]);
    h = mix64(h ^ (uint64_t)bd);
    h = mix64(h ^ (uint64_t)noff);
    for (int32_t j = 0; j < noff; j++) h = mix64(h ^ (uint64_t)P.scr_off[t.base + j]);
    h = mix64(h ^ (uint64_t)ndrop);
    for (int32_t j = 0; j < ndrop; j++) h = mix64(h ^ (uint64_t)P.scr_drop[t.base + j]);
    h = mix64(h ^ (uint64_t)npre);
    for (int32_t j = 0; j < npre; j++) h = mix64(h ^ (uint64_t)P.scr_pre[t.base + j]);
    h = mix64(h ^ (uint64_t)lat);
    I.hash = h;
  }
  __syncwarp();
}

// --------------------------------------------------------------------------- LP formation ---
__device__ void form_lp(const SimP& P, SInst* SI, int k, Tr& t, int64_t T, KI* sbuf) {
  SInst& I = SI[k];
  const int lane = lane_id();
  const int64_t o = ioff(P, k, t);
  const int32_t ndrop = drop_step(P, I, k, t, T);
  const int32_t npre = decode_prep(P, I, k, t);
  t.evals += I.wq_len;
  const int64_t Bd = I.ds_len;
  const int64_t sl = Bd ? ds_ctx_sum(P, I, k, t) : 0;
  // budgets (G22)
  const int64_t N = P.lp_tok, M = I.kv_free, Rb = P.lp_max - Bd;
  int64_t C = INF64;
  if (Bd) {
    const int64_t d = lat_us(P.md, 0, 0, 0, 0, (uint64_t)Bd, (uint64_t)sl);
    if (d < 0) atomicOr(P.err, ERR_RANGE);
    C = t.tbt - d;
  }
  // Algorithm 1: K smallest (key, id) of the waiting queue, sorted (line 3) ...
  const int32_t len = I.wq_len;
  int32_t nadm = 0;
  uint64_t sp = 0, sp2 = 0, spc = 0;
  KI last = ki_inf();
  if (len > 0) {
    TopKStream<KPL> st;
    st.init(sbuf);
    for (int32_t c = 0; c < len; c += 32) {
      const int32_t j = c + lane;
      const bool v = j < len;
      KI x = ki_inf();
      if (v) x = KI{P.wq_key[o + j], P.wq_id[o + j]};
      st.push(x, v);
    }
    st.finish();
    __syncwarp();
    // ... lines 5-13 as a strict prefix-sum scan over the sorted candidates
    int64_t ct = 0, cb = 0, cc = 0;
    bool go = true;
#pragma unroll
    for (int r = 0; r < KPL; r++) {
      const KI e = st.top.a[r];
      const bool valid = e.i != INF32;
      const int64_t g = t.base + (valid ? e.i : 0);
      const int32_t p = valid ? P.rq_eff[g] : 0;
      const int64_t pf = valid ? pf_of(P, p) : 0;
      const int64_t bl = valid ? blk_of(P, p) : 0;
      const int64_t St = ct + warp_incl_scan((int64_t)p);
      const int64_t Sb = cb + warp_incl_scan(bl);
      const int64_t Sc = cc + warp_incl_scan(pf);
      const int pos = r * 32 + lane;
      const bool ok = go && valid && St < N && Sb < M && Sc < C && pos < Rb;
      const uint32_t m = __ballot_sync(FULL, ok);
      const int cnt = (m == FULL) ? 32 : (__ffs(~m) - 1);
      const bool adm = go && lane < cnt;
      if (adm) {
        admit_req(P, g, k, T);
        P.bp_id[o + pos] = e.i;
        const uint64_t q = (uint64_t)p;
        sp += q;
        sp2 += q * q;
        spc += q * ceil_div_u(q, P.md.b);
      }
      nadm += go ? cnt : 0;
      if (cnt < 32) go = false;
      ct = __shfl_sync(FULL, St, 31);
      cb = __shfl_sync(FULL, Sb, 31);
      cc = __shfl_sync(FULL, Sc, 31);
    }
    if (nadm > 0) last = ki_shfl(st.top.a[(nadm - 1) >> 5], (nadm - 1) & 31);
    sp = warp_sum(sp);
    sp2 = warp_sum(sp2);
    spc = warp_sum(spc);
  }
  // admitted KV blocks: sum_j ceil((p_j + 1)/bs)
  int64_t used = 0;
  for (int32_t j = lane; j < nadm; j += 32) used += blk_of(P, P.rq_eff[t.base + P.bp_id[o + j]]);
  used = warp_sum(used);
  // offload (§5.3, G24) + queue compaction in one pass; the admitted set is exactly the entries
  // at or before `last` in (key, id) order
  int32_t noff = 0;
  if (len > 0 && (nadm > 0 || P.offl)) {
    int32_t out = 0;
    for (int32_t c = 0; c < len; c += 32) {
      const int32_t j = c + lane;
      const bool v = j < len;
      KI x = ki_inf();
      bool adm = false, off = false;
      if (v) {
        x = KI{P.wq_key[o + j], P.wq_id[o + j]};
        adm = nadm > 0 && !ki_less(last, x);
        if (!adm && P.offl) {
          const int64_t g = t.base + x.i;
          const uint32_t f = P.rq_fl[g];
          off = !(f & (F_EVER | F_ONHP)) &&
                P.rq_dl[g] - T <= pf_of(P, P.rq_eff[g]) + P.W + P.margin;
        }
      }
      const bool keep = v && !adm && !off;
      const uint32_t mk = __ballot_sync(FULL, keep), mo = __ballot_sync(FULL, off);
      __syncwarp();
      if (keep) { const int32_t q = out + __popc(mk & lanemask_lt()); P.wq_id[o + q] = x.i; P.wq_key[o + q] = x.k; }
      if (off) P.scr_off[t.base + noff + __popc(mo & lanemask_lt())] = x.i;
      out += __popc(mk);
      noff += __popc(mo);
      __syncwarp();
    }
    if (lane == 0) I.wq_len = out;
    __syncwarp();
  }
  if (lane == 0) I.kv_free -= (int32_t)used;
  __syncwarp();
  // dispatch offloads round-robin over the HPs, ascending id
  for (int32_t j = 0; j < noff; j++) {
    const int32_t id = P.scr_off[t.base + j];
    const int64_t g = t.base + id;
    if (lane == 0) P.rq_fl[g] |= (F_ONHP | F_OFFL);
    __syncwarp();
    const int h = P.n_lp + t.rr_hp;
    t.rr_hp = (t.rr_hp + 1) % P.n_hp;
    if (P.delay == 0) {
      wq_insert_sorted(P, SI[h], h, t, id);
    } else {
      if (lane == 0) {
        P.fl_t[t.base + t.fl_tail] = T + P.delay;
        P.fl_req[t.base + t.fl_tail] = id;
        P.fl_hp[t.base + t.fl_tail] = h;
      }
      __syncwarp();
      t.fl_tail++;
    }
  }
  // batch (§5.4): decodes piggybacked with the admitted prefills
  const bool nonempty = nadm > 0 || Bd > 0;
  int64_t l = 0;
  if (nonempty) {
    l = lat_us(P.md, (uint64_t)nadm, sp, sp2, spc, (uint64_t)Bd, (uint64_t)sl);
    if (l < 0) atomicOr(P.err, ERR_RANGE);
    if (lane == 0) {
      I.end = T + l;
      I.busy = 1;
      I.batch_dec = Bd > 0;
      I.bp_len = nadm;
    }
    __syncwarp();
    t.decisions++;
  }
  if (nonempty || noff || ndrop || npre) digest_log(P, I, k, t, T, nadm, nonempty ? Bd : 0, noff, ndrop, npre, l);
}

// --------------------------------------------------------------------------- HP formation ---
// FCFS prefill-first under the (elastic) token limit (G27-G28).
__device__ int32_t hp_prefill(const SimP& P, SInst& I, int k, const Tr& t, int64_t T,
                              uint64_t& sp, uint64_t& sp2, uint64_t& spc) {
  const int lane = lane_id();
  const int64_t o = ioff(P, k, t);
  int64_t limit = P.hp_tok;
  if (P.elastic) {
    const int64_t mean = I.hist_cnt ? I.hist_sum / I.hist_cnt : (int64_t)P.hist_def;
    const int64_t avail = (int64_t)I.kv_free * P.bs - mean * ((int64_t)I.ds_len + 1);
    if (10 * avail > (int64_t)I.kv_total * P.bs) limit = P.hp_tok + avail;
  }
  const int32_t len = I.wq_len;
  const int64_t kvf = I.kv_free;
  int64_t ct = 0, cb = 0;
  int32_t nadm = 0;
  sp = sp2 = spc = 0;
  for (int32_t c = 0; c < len; c += 32) {
    const int32_t j = c + lane;
    const bool v = j < len;
    int32_t id = 0, p = 0;
    if (v) { id = P.wq_id[o + j]; p = P.rq_eff[t.base + id]; }
    const int64_t bl = v ? blk_of(P, p) : 0;
    const int64_t St = ct + warp_incl_scan((int64_t)p);
    const int64_t Sb = cb + warp_incl_scan(bl);
    const bool ok = v && ((j == 0) ? (bl <= kvf) : (St <= limit && Sb <= kvf));
    const uint32_t m = __ballot_sync(FULL, ok);
    const int cnt = (m == FULL) ? 32 : (__ffs(~m) - 1);
    if (lane < cnt) {
      admit_req(P, t.base + id, k, T);
      P.bp_id[o + j] = id;
      const uint64_t q = (uint64_t)p;
      sp += q;
      sp2 += q * q;
      spc += q * ceil_div_u(q, P.md.b);
    }
    nadm += cnt;
    if (cnt < 32) break;
    ct = __shfl_sync(FULL, St, 31);
    cb = __shfl_sync(FULL, Sb, 31);
  }
  sp = warp_sum(sp);
  sp2 = warp_sum(sp2);
  spc = warp_sum(spc);
  if (nadm == 0) return 0;
  int64_t used = 0;
  for (int32_t j = lane; j < nadm; j += 32) used += blk_of(P, P.rq_eff[t.base + P.bp_id[o + j]]);
  used = warp_sum(used);
  // remove the admitted prefix
  for (int32_t c = 0; c < len - nadm; c += 32) {
    const int32_t j = c + lane;
    const bool v = j < len - nadm;
    int32_t xi = 0;
    int64_t xk = 0;
    if (v) { xi = P.wq_id[o + nadm + j]; xk = P.wq_key[o + nadm + j]; }
    __syncwarp();
    if (v) { P.wq_id[o + j] = xi; P.wq_key[o + j] = xk; }
    __syncwarp();
  }
  if (lane == 0) { I.wq_len = len - nadm; I.kv_free -= (int32_t)used; }
  __syncwarp();
  return nadm;
}

__device__ void form_hp(const SimP& P, SInst* SI, int k, Tr& t, int64_t T) {
  SInst& I = SI[k];
  const int lane = lane_id();
  const int32_t ndrop = drop_step(P, I, k, t, T);
  t.evals += I.wq_len;
  uint64_t sp = 0, sp2 = 0, spc = 0;
  int32_t nadm = 0, npre = 0;
  int64_t bd = 0, sl = 0;
  bool batch = false;
  if (I.wq_len > 0) { nadm = hp_prefill(P, I, k, t, T, sp, sp2, spc); batch = nadm > 0; }
  if (!batch && I.ds_len > 0) {
    npre = decode_prep(P, I, k, t);
    if (I.ds_len > 0) {
      batch = true;
      bd = I.ds_len;
      sl = ds_ctx_sum(P, I, k, t);
    } else if (I.wq_len > 0) {
      nadm = hp_prefill(P, I, k, t, T, sp, sp2, spc);
      batch = nadm > 0;
    }
  }
  int64_t l = 0;
  if (batch) {
    l = bd ? lat_us(P.md, 0, 0, 0, 0, (uint64_t)bd, (uint64_t)sl)
           : lat_us(P.md, (uint64_t)nadm, sp, sp2, spc, 0, 0);
    if (l < 0) atomicOr(P.err, ERR_RANGE);
    if (lane == 0) {
      I.end = T + l;
      I.busy = 1;
      I.batch_dec = bd > 0;
      I.bp_len = bd ? 0 : nadm;
    }
    __syncwarp();
    t.decisions++;
  }
  if (batch || ndrop || npre) digest_log(P, I, k, t, T, bd ? 0 : nadm, bd, 0, ndrop, npre, l);
}

// ------------------------------------------------------------------ phase A: batch completion --
__device__ void finish_req(const SimP& P, int64_t g, int64_t T) {
  P.done[g] = T;
  set_state(P, g, 1u);
}

__device__ void complete(const SimP& P, SInst& I, int k, const Tr& t, int64_t T) {
  const int lane = lane_id();
  const int64_t o = ioff(P, k, t);
  int64_t freed = 0, hsum = 0;
  int32_t hcnt = 0, tkd = 0;
  int32_t dlen = I.ds_len;
  if (I.batch_dec) {
    int32_t out = 0;
    for (int32_t c = 0; c < dlen; c += 32) {
      const int32_t j = c + lane;
      const bool v = j < dlen;
      int32_t id = 0, ctx = 0, held = 0, rem = 0;
      bool fin = false;
      if (v) {
        id = P.ds_id[o + j]; ctx = P.ds_ctx[o + j] + 1; held = P.ds_held[o + j]; rem = P.ds_rem[o + j] - 1;
        fin = rem == 0;
        if (fin) {
          const int64_t g = t.base + id;
          finish_req(P, g, T);
          freed += held;
          if (I.hp) { hsum += P.ol[g]; hcnt++; if (P.rq_fl[g] & F_TICK) tkd++; }
        }
      }
      const uint32_t mk = __ballot_sync(FULL, v && !fin);
      __syncwarp();
      if (v && !fin) {
        const int32_t q = out + __popc(mk & lanemask_lt());
        P.ds_id[o + q] = id; P.ds_ctx[o + q] = ctx; P.ds_held[o + q] = held; P.ds_rem[o + q] = rem;
      }
      out += __popc(mk);
      __syncwarp();
    }
    dlen = out;
  }
  const int32_t blen = I.bp_len;
  for (int32_t c = 0; c < blen; c += 32) {
    const int32_t j = c + lane;
    const bool v = j < blen;
    bool stay = false;
    int32_t id = 0, ctx = 0, held = 0, rem = 0;
    if (v) {
      id = P.bp_id[o + j];
      const int64_t g = t.base + id;
      const int32_t eff = P.rq_eff[g], p = P.pl[g], out_len = P.ol[g];
      const int32_t gen = eff - p + 1;  // tokens generated after this prefill
      if (P.first[g] < 0) P.first[g] = T;
      held = blk_of(P, eff);
      if (gen == out_len) {
        finish_req(P, g, T);
        freed += held;
        if (I.hp) { hsum += out_len; hcnt++; if (P.rq_fl[g] & F_TICK) tkd++; }
      } else {
        stay = true;
        ctx = p + gen;
        rem = out_len - gen;
      }
    }
    const uint32_t ms = __ballot_sync(FULL, stay);
    if (stay) {
      const int32_t q = dlen + __popc(ms & lanemask_lt());
      P.ds_id[o + q] = id; P.ds_ctx[o + q] = ctx; P.ds_held[o + q] = held; P.ds_rem[o + q] = rem;
    }
    dlen += __popc(ms);
  }
  freed = warp_sum(freed);
  hsum = warp_sum(hsum);
  hcnt = warp_sum(hcnt);
  tkd = warp_sum(tkd);
  __syncwarp();
  if (lane == 0) {
    I.ds_len = dlen;
    I.kv_free += (int32_t)freed;
    I.hist_sum += hsum;
    I.hist_cnt += hcnt;
    I.tk_live -= tkd;
    I.bp_len = 0;
    I.batch_dec = 0;
    I.busy = 0;
  }
  __syncwarp();
}

// --------------------------------------------------------------------- controller routing ---
__device__ void route(const SimP& P, SInst* SI, Tr& t, int32_t id) {
  if (P.tickets) {
    for (int h = P.n_lp; h < P.K; h++) {
      if (SI[h].ticket) {
        if (lane_id() == 0) {
          SI[h].ticket = 0;
          SI[h].tk_live += 1;
          P.rq_fl[t.base + id] |= (F_TICK | F_ONHP);
        }
        __syncwarp();
        wq_append(P, SI[h], h, t, id);  // the newest arrival has the largest id: stays sorted
        return;
      }
    }
  }
  wq_append(P, SI[t.rr_lp], t.rr_lp, t, id);
  t.rr_lp = (t.rr_lp + 1) % P.n_lp;
}

__global__ void __launch_bounds__(SW * 32) sim_kernel(SimP P) {
  __shared__ SInst s_inst[SW][MAXI];
  __shared__ KI s_buf[SW][64];
  __shared__ int s_trace[SW];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  SInst* SI = s_inst[w];
  while (true) {
    if (lane == 0) s_trace[w] = atomicAdd(P.next_trace, 1);
    __syncwarp();
    const int trace = s_trace[w];
    __syncwarp();
    if (trace >= P.T) break;
    Tr t;
    t.base = P.off[trace];
    t.n = P.off[trace + 1] - t.base;
    t.tbt = P.tbt[trace];
    t.next = t.fl_head = t.fl_tail = t.decisions = t.evals = 0;
    t.rr_lp = t.rr_hp = 0;
    const int64_t ttft = P.ttft[trace];
    for (int64_t i = lane; i < t.n; i += 32) {
      const int64_t g = t.base + i;
      P.rq_dl[g] = P.arr[g] + (P.rttft ? P.rttft[g] : ttft);
      P.rq_eff[g] = P.pl[g];
      P.rq_fl[g] = 0xffu << INST_SHIFT;
      P.first[g] = -1;
      P.done[g] = -1;
      P.pstart[g] = -1;
    }
    if (lane < P.K) {
      SInst& I = SI[lane];
      I.hp = lane >= P.n_lp;
      I.kv_total = I.kv_free = I.hp ? P.kv_hp : P.kv_lp;
      I.end = 0; I.hist_sum = 0; I.hash = 0;
      I.wq_len = I.ds_len = I.bp_len = I.hist_cnt = 0;
      I.busy = I.batch_dec = I.tk_live = 0;
      I.ticket = (I.hp && P.tickets) ? 1 : 0;  // issued at t = 0 (G29)
    }
    __syncwarp();
    while (true) {
      int64_t T = INF64;
      if (t.next < t.n) T = P.arr[t.base + t.next];
      int64_t te = INF64;
      if (lane < P.K && SI[lane].busy) te = SI[lane].end;
      te = warp_min(te);
      T = te < T ? te : T;
      if (t.fl_head < t.fl_tail) {
        const int64_t tf = P.fl_t[t.base + t.fl_head];
        T = tf < T ? tf : T;
      }
      if (T == INF64) {
        const bool stuck = lane < P.K && (SI[lane].wq_len > 0 || SI[lane].ds_len > 0);
        if (__any_sync(FULL, stuck) && lane == 0) atomicOr(P.err, ERR_INVARIANT);
        break;
      }
      // A. completions in instance order
      for (int k = 0; k < P.K; k++)
        if (SI[k].busy && SI[k].end == T) complete(P, SI[k], k, t, T);
      // B. offload deliveries (FIFO = time order)
      while (t.fl_head < t.fl_tail && P.fl_t[t.base + t.fl_head] == T) {
        const int32_t id = P.fl_req[t.base + t.fl_head];
        const int h = P.fl_hp[t.base + t.fl_head];
        wq_insert_sorted(P, SI[h], h, t, id);
        t.fl_head++;
      }
      // C. arrivals, ascending id
      while (t.next < t.n && P.arr[t.base + t.next] == T) {
        route(P, SI, t, (int32_t)t.next);
        t.next++;
      }
      // D. formations of idle instances, LPs before HPs
      for (int k = 0; k < P.K; k++) {
        if (SI[k].busy) continue;
        if (SI[k].hp) form_hp(P, SI, k, t, T);
        else form_lp(P, SI, k, t, T, s_buf[w]);
      }
      // E. tickets (G29)
      if (P.tickets) {
        if (lane >= P.n_lp && lane < P.K) {
          SInst& I = SI[lane];
          if (!I.ticket && I.wq_len == 0 && I.tk_live == 0) I.ticket = 1;
        }
        __syncwarp();
      }
    }
    // outputs
    for (int64_t i = lane; i < t.n; i += 32) {
      const int64_t g = t.base + i;
      const uint32_t f = P.rq_fl[g];
      uint32_t st = (f >> ST_SHIFT) & 3u;
      st |= (f & F_OFFL) ? 4u : 0u;
      st |= (f & F_TICK) ? 8u : 0u;
      st |= ((f >> INST_SHIFT) & 0xffu) << 4;
      st |= ((f >> NPRE_SHIFT) & 0xffffu) << 12;
      P.status[g] = st;
    }
    if (lane == 0) {
      uint64_t d = 0;
      for (int k = 0; k < P.K; k++) d = mix64(d ^ SI[k].hash);
      P.digest[trace] = d;
      if (P.decisions) P.decisions[trace] = t.decisions;
      if (P.evals) P.evals[trace] = t.evals;
    }
    __syncwarp();
  }
}

// liveness / layout validation (ASC_E_CONFIG / ASC_E_INVAL before simulating)
__global__ void validate_traces(SimP P, int64_t R) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < R;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = P.pl[g], o = P.ol[g];
    if (p < 1 || o < 1 || (int64_t)p + o > P.lp_tok) atomicOr(P.err, 8);
    const int64_t nb = ((int64_t)p + o + P.bs - 1) / P.bs;
    const int64_t kvmin = P.n_hp ? (P.kv_lp < P.kv_hp ? P.kv_lp : P.kv_hp) : P.kv_lp;
    if (nb >= kvmin) atomicOr(P.err, 8);
    if (g > 0 && P.arr[g] < P.arr[g - 1]) {
      // arrivals must be non-decreasing inside a trace (a trace boundary may step down)
      int64_t lo = 0, hi = P.T;  // find trace of g: largest t with off[t] <= g
      while (hi - lo > 1) { const int64_t mid = (lo + hi) >> 1; if (P.off[mid] <= g) lo = mid; else hi = mid; }
      if (P.off[lo] != g) atomicOr(P.err, ERR_INVAL);
    }
  }
}

// a8: goodput numerator/denominator per trace
__global__ void goodput_kernel(int32_t T, const int64_t* off, const int64_t* arr, const int32_t* ol,
                               const int64_t* ttft, const int64_t* tbt, const int64_t* rttft,
                               const int64_t* first, const int64_t* done, const uint32_t* status,
                               uint64_t* good, uint64_t* total, int* err) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = w; t < T; t += nw) {
    const int64_t lo = off[t], hi = off[t + 1];
    const int64_t tt = ttft[t], tb = tbt[t];
    uint64_t g = 0;
    for (int64_t i = lo + lane; i < hi; i += 32) {
      if ((__ldcs(status + i) & 3u) != 1u) continue;
      const int64_t f = __ldcs(first + i);
      const int64_t slo = rttft ? rttft[i] : tt;
      if (f - __ldcs(arr + i) > slo) continue;
      const int32_t o = __ldcs(ol + i);
      if (o > 1 && __ldcs(done + i) - f > tb * (int64_t)(o - 1)) continue;
      g++;
    }
    g = warp_sum(g);
    if (lane == 0) {
      good[t] = g;
      total[t] = (uint64_t)(hi - lo);
      if (hi == lo) atomicOr(err, 16);
    }
  }
}

}  // namespace

namespace asc {

asc_status launch_simulate(asc_ctx* c, const asc_traces* tr, asc_outcomes* out, int64_t R) {
  const asc_config& cf = c->cfg;
  const int K = cf.topo.n_lp + cf.topo.n_hp;
  const int32_t T = tr->T;
  size_t need = (size_t)R * (8 + 4 + 4) + (size_t)K * R * (8 + 4 + 16 + 4) + (size_t)R * 12 +
                (cf.flags.offload_delay_us ? (size_t)R * 16 : 0) + 64 * 1024;
  asc_status st = ensure_ws(c, need);
  if (st) return st;
  Arena ar{c->ws, c->ws_cap};
  SimP P;
  P.md = c->md;
  P.pf_tab = c->d_pf_tab;
  P.pt = c->pt_size;
  P.n_lp = cf.topo.n_lp; P.n_hp = cf.topo.n_hp; P.K = K; P.bs = cf.topo.block_tokens;
  P.lp_max = cf.topo.lp_max_batch; P.lp_tok = cf.topo.lp_token_budget; P.hp_tok = cf.topo.hp_token_budget;
  P.policy = cf.flags.policy;
  P.offl = (cf.flags.offload && cf.topo.n_hp >= 1) ? 1 : 0;
  P.tickets = (cf.flags.tickets && cf.topo.n_hp >= 1) ? 1 : 0;
  P.elastic = cf.flags.elastic; P.drop = cf.flags.drop; P.hist_def = cf.flags.hist_default_tokens;
  P.kv_lp = cf.topo.kv_blocks_lp; P.kv_hp = cf.topo.kv_blocks_hp;
  P.W = c->w_hp; P.margin = cf.flags.offload_margin_us; P.delay = cf.flags.offload_delay_us;
  P.T = T; P.off = tr->trace_off; P.arr = tr->arrival_us; P.pl = tr->prompt_len; P.ol = tr->output_len;
  P.ttft = tr->ttft_slo_us; P.tbt = tr->tbt_slo_us; P.rttft = tr->req_ttft_slo_us;
  P.first = out->first_token_us; P.done = out->done_us; P.pstart = out->prefill_start_us;
  P.status = out->status; P.digest = out->digest; P.decisions = out->decisions; P.evals = out->evaluations;
  P.R = R;
  P.rq_dl = ar.take<int64_t>(R);
  P.rq_eff = ar.take<int32_t>(R);
  P.rq_fl = ar.take<uint32_t>(R);
  P.wq_key = ar.take<int64_t>((size_t)K * R);
  P.wq_id = ar.take<int32_t>((size_t)K * R);
  P.ds_id = ar.take<int32_t>((size_t)K * R);
  P.ds_ctx = ar.take<int32_t>((size_t)K * R);
  P.ds_held = ar.take<int32_t>((size_t)K * R);
  P.ds_rem = ar.take<int32_t>((size_t)K * R);
  P.bp_id = ar.take<int32_t>((size_t)K * R);
  P.scr_drop = ar.take<int32_t>(R);
  P.scr_pre = ar.take<int32_t>(R);
  P.scr_off = ar.take<int32_t>(R);
  if (cf.flags.offload_delay_us) {
    P.fl_t = ar.take<int64_t>(R);
    P.fl_req = ar.take<int32_t>(R);
    P.fl_hp = ar.take<int32_t>(R);
  } else {
    P.fl_t = nullptr; P.fl_req = nullptr; P.fl_hp = nullptr;
  }
  P.next_trace = ar.take<int>(1);
  P.err = c->d_err;
  cudaStream_t sm = c->stream;
  int64_t launches = 0;
  if (R > 0) {
    const int64_t gb = (R + 255) / 256;
    validate_traces<<<(unsigned)(gb < 4096 ? gb : 4096), 256, 0, sm>>>(P, R);
    launches++;
    asc_status v = collect_errors(c, "simulate_batch validation");
    if (v) return v;
  }
  cudaMemsetAsync(P.next_trace, 0, sizeof(int), sm);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  int64_t blocks = ((int64_t)T + SW - 1) / SW;
  const int64_t cap = (int64_t)sms * 16;
  if (blocks > cap) blocks = cap;
  if (blocks > 0) {
    cudaEventRecord(c->ev0, sm);
    sim_kernel<<<(unsigned)blocks, SW * 32, 0, sm>>>(P);
    cudaEventRecord(c->ev1, sm);
    c->timed = true;
    launches++;
  }
  c->last_kernel_launches = launches;
  return cuda_check(c, cudaGetLastError(), "simulate launch");
}

asc_status launch_goodput(asc_ctx* c, const asc_traces* tr, const asc_outcomes* out,
                          uint64_t* good, uint64_t* total) {
  const int32_t T = tr->T;
  if (T <= 0) return ASC_OK;
  int64_t blocks = ((int64_t)T * 32 + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  cudaEventRecord(c->ev0, c->stream);
  goodput_kernel<<<(unsigned)blocks, 256, 0, c->stream>>>(
      T, tr->trace_off, tr->arrival_us, tr->output_len, tr->ttft_slo_us, tr->tbt_slo_us,
      tr->req_ttft_slo_us, out->first_token_us, out->done_us, out->status, good, total, c->d_err);
  cudaEventRecord(c->ev1, c->stream);
  c->timed = true;
  c->last_kernel_launches = 1;
  return cuda_check(c, cudaGetLastError(), "goodput launch");
}

}  // namespace asc
