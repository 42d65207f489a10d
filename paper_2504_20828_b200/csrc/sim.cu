// sim.cu — asc_simulate_batch: the batched discrete-event step loop (with
// rows a1-a6 inlined per formation) and asc_goodput (row a8).
//
// One warp owns one trace at a time (traces are handed out by an atomic counter so long traces
// do not serialise a static partition).  Per-trace state stays resident on the GPU:
//   per request  (HBM)  : deadline (int64), effective prompt (int32), flag word (uint32)
//   per instance (HBM)  : waiting queue (key, id) with time-invariant keys, the
//                         running batch's prefill ids
//   per instance (SMEM) : scalars (end = INF when idle, kv_free, ticket, history, running Σl̂,
//                         pending KV growth, digest) and the first 128 decode slots
//                         {id, l̂, remaining, held | (l̂ mod bs)<<22 | pending<<31}
//                         (LP decode sets never exceed 128 = P:371; HP slots beyond spill to HBM)
//   per trace    (HBM)  : drop / eviction / offload scratch lists and the in-flight offload ring
// A decode step — by far the most frequent decision — costs one pass over the decode slots in
// shared memory (the completion pass also precomputes the next formation's block growth and
// Σl̂, with no integer division), one closed-form decode cost + fp64 evaluation of Eq. 4-5, and
// an 8-lane digest update.  Rare paths (admission with a non-empty queue, eviction, drops, HP
// prefill, offload dispatch, prefill completions) are __noinline__ so the hot loop stays small.
// The event order is the canonical A-E phase order of DESIGN.md §2.
#include <cstdlib>
#include <mutex>
#include "asc_internal.h"

using namespace asc;

namespace {

constexpr int KPL = 4;
constexpr int SW = 4;      // warps (traces in flight) per CTA
#ifndef ASC_DCAP
#define ASC_DCAP 64
#endif
constexpr int DCAP = ASC_DCAP;  // decode slots per instance kept in shared memory
constexpr uint64_t GOLD = 0x9E3779B97F4A7C15ull;
constexpr uint64_t GOLD2 = 0xD1B54A32D192ED03ull;  // formation-index key of the instance digest

enum : uint32_t { F_EVER = 1u, F_ONHP = 2u, F_TICK = 4u, F_OFFL = 8u };
constexpr uint32_t ST_SHIFT = 4, INST_SHIFT = 8, NPRE_SHIFT = 16;
// decode slot .w: bits 0-21 blocks held (before pending growth), 22-30 l̂ mod bs, 31 pending
constexpr int32_t HELD_MASK = (1 << 22) - 1;
constexpr int R_SHIFT = 22;
constexpr int32_t PEND = (int32_t)0x80000000;

struct SInst {
  int64_t end;               // end of the running batch, INF64 when idle
  int64_t hist_sum, ctx_sum;
  uint64_t hash, nrec;       // instance digest and number of recorded formations
  int32_t kv_free, kv_total, wq_len, ds_len, bp_len, hist_cnt, need_sum;
  int32_t batch_dec, ticket, tk_live, hp, papp;
  int32_t wq_head;           // the waiting queue occupies [wq_head, wq_head + wq_len) of the region
};

struct SimP {
  Model md;
  const int64_t* pf_tab;
  int32_t pt;
  int32_t n_lp, n_hp, K, bs, lp_max, lp_tok, hp_tok, policy, offl, tickets, elastic, drop, hist_def;
  uint64_t bs_m;  // ceil(2^38 / bs): x / bs = (x * bs_m) >> 38 exactly for 0 <= x < 2^25 (bs <= 512)
  uint64_t ab_m;  // ceil(2^38 / b) for the attention block b (ceilb), used when ab_fast
  int32_t ab_fast;  // b <= 4096: (x * ab_m) >> 38 == x / b for every x < 2^25 + b
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
  int4* ds_g;  // decode-slot overflow (slot index >= DCAP)
  int32_t* bp_id;
  int32_t *scr_drop, *scr_pre, *scr_off, *scr_tmp;
  int64_t* fl_t;
  int32_t *fl_req, *fl_hp;
  int* err;
  int* next_trace;
  int32_t pw, o_sd, o_si, o_ts;  // per-warp shared-memory layout (bytes)
  int32_t mode;                  // asc_scheduler (0 Ascendra, 1 vLLM-like, 2 Sarathi-like)
  int32_t chunk_tok;             // Sarathi-like per-batch token budget
  int32_t* rq_cdone;             // Sarathi-like: prompt tokens prefilled (after the running chunk)
  const int32_t *tr_nlp, *tr_nhp;  // optional per-trace topology (row f3)
  int32_t look;                    // offload rule 1: look-ahead (G50)
  int32_t kw0, kw1, kw2;           // ASC_POLICY_WEIGHTED weights (G51)
  const int64_t* rq_koff;          // optional per-request value-function offsets (G51)
  // decision snapshots (asc_arm_snapshots; sn_hdr == nullptr when not armed)
  int64_t *sn_hdr, *sn_cnt, *sn_dl;
  int32_t *sn_ids, *sn_eff, *sn_out;
  uint8_t* sn_fl;
  int32_t sn_trace, sn_inst, sn_max;
  int64_t sn_every, sn_ecap, sn_ocap;
};

// The launch parameters live in the constant bank (one copy per device, written before each launch
// under the per-device lock in launch_simulate): every out-of-line device function reads them as
// constant operands, with no pointer to reload after stores.
__constant__ SimP P;


struct TS {  // per-trace controller state (shared memory, one per warp)
  int32_t rr_lp, rr_hp, fl_head, fl_tail;
  int32_t n_lp, n_hp, K, sw;  // the trace's subgroup topology; sw: 1 offload, 2 tickets
  int64_t base, n, tbt;  // the trace's first request, its size and its TBT SLO
};

// Per-warp trace context.  Empty: every member is recomputed from the warp index and the
// constant-bank layout, so nothing is passed in registers across the out-of-line calls and the
// compiler sees shared-memory addresses (LDS/STS, not generic loads).
struct Wp {
  __device__ __forceinline__ unsigned char* mine() const {
    extern __shared__ __align__(16) unsigned char smem[];
    return smem + (threadIdx.x >> 5) * P.pw;
  }
  __device__ __forceinline__ KI* buf() const { return reinterpret_cast<KI*>(mine()); }
  __device__ __forceinline__ int4* sd() const { return reinterpret_cast<int4*>(mine() + P.o_sd); }
  __device__ __forceinline__ SInst* SI() const { return reinterpret_cast<SInst*>(mine() + P.o_si); }
  __device__ __forceinline__ TS* ts() const { return reinterpret_cast<TS*>(mine() + P.o_ts); }
  __device__ __forceinline__ int64_t base() const { return ts()->base; }
  __device__ __forceinline__ int64_t n() const { return ts()->n; }
  __device__ __forceinline__ int64_t tbt() const { return ts()->tbt; }
  __device__ __forceinline__ int nlp() const { return ts()->n_lp; }
  __device__ __forceinline__ int nhp() const { return ts()->n_hp; }
  __device__ __forceinline__ int K() const { return ts()->K; }
  __device__ __forceinline__ bool offl() const { return ts()->sw & 1; }
  __device__ __forceinline__ bool tickets() const { return ts()->sw & 2; }
};

// Out-of-line copies of the rarely taken latency evaluations: inlined, each call site would carry
// its own copy of the integer moments, the wrap guard and the fp64 regression, and the event loop's
// hot code would outgrow the instruction cache (the kernel is instruction-fetch bound).
__device__ __noinline__ int64_t pf_slow(int32_t p) {  // prompts beyond the per-ctx table
  const int64_t v = prefill_lat(P.md, (uint64_t)p);
  if (v < 0) { atomicOr(P.err, ERR_RANGE); return INT32_MAX; }
  return v;
}
__device__ __forceinline__ int64_t pf_of(int32_t p) {
  return p < P.pt ? __ldg(P.pf_tab + p) : pf_slow(p);
}
__device__ __noinline__ int64_t lat_dec_call(int64_t Bd, int64_t sl) {  // decode-only batch, Eq. 4-5
  return lat_decode(P.md, (uint64_t)Bd, (uint64_t)sl);
}
__device__ __noinline__ int64_t lat_batch(uint64_t nadm, uint64_t sp, uint64_t sp2, uint64_t spc, uint64_t Bd,
                                         uint64_t sl) {  // hybrid batch from its moments, Eq. 3-5
  return lat_us(P.md, nadm, sp, sp2, spc, Bd, sl);
}
// division by the block size without a division sequence: with m = ceil(2^38 / bs) = (2^38 + e) / bs,
// 0 <= e < bs <= 512, x * m / 2^38 = x / bs + x * e / (bs * 2^38) and x * e < 2^38 for x < 2^29, so the
// error term stays below 1 / bs and never crosses an integer; every argument here is a token count
// or event index below lp_token_budget + bs < 2^25 (validated), so x * m < 2^63 does not overflow
__device__ __forceinline__ int32_t divb(int32_t x) { return (int32_t)(((uint64_t)(uint32_t)x * P.bs_m) >> 38); }
__device__ __forceinline__ int32_t modb(int32_t x) { return x - divb(x) * P.bs; }
__device__ __forceinline__ int32_t blk_of(int32_t eff) { return divb(eff + P.bs); }
// ceil(u / b), b = the attention block (App. A.1, G15); u < 2^25 (a token count)
__device__ __forceinline__ uint64_t ceilb(uint64_t u) {
  const uint32_t x = (uint32_t)u + (uint32_t)P.md.b - 1u;
  return P.ab_fast ? (uint64_t)(((uint64_t)x * P.ab_m) >> 38) : (uint64_t)(x / (uint32_t)P.md.b);
}

// time-invariant priority key of request gid with effective prompt eff (DESIGN.md §2 Keys)
__device__ __forceinline__ int64_t key_of(int64_t gid, int32_t eff) {
  int64_t k;
  switch (P.policy) {
    case 0: k = P.rq_dl[gid] - pf_of(eff); break;
    case 1: k = P.rq_dl[gid]; break;
    case 2: k = pf_of(eff); break;
    case 3: k = -pf_of(eff); break;
    case 5: k = (int64_t)P.kw0 * P.rq_dl[gid] + (int64_t)P.kw1 * pf_of(eff) + (int64_t)P.kw2 * P.arr[gid]; break;
    default: k = P.arr[gid]; break;
  }
  return P.rq_koff ? k + P.rq_koff[gid] : k;  // service-class offset (G51)
}

__device__ __forceinline__ int64_t ioff(int k, Wp w) { return (int64_t)k * P.R + w.base(); }
__device__ __forceinline__ int4* slotp(Wp w, int k, int32_t j) {
  return j < DCAP ? (w.sd() + k * DCAP + j) : (P.ds_g + (int64_t)k * P.R + w.base() + j);
}
__device__ __forceinline__ void set_state(int64_t g, uint32_t st) {
  const uint32_t f = P.rq_fl[g];
  P.rq_fl[g] = (f & ~(3u << ST_SHIFT)) | (st << ST_SHIFT);
}

// ------------------------------------------------------------------------------- digest ------
#ifdef ASC_MIX1
__device__ __forceinline__ uint64_t mixi(uint64_t x) { return (x ^ (x >> 32)) * 0xbf58476d1ce4e5b9ull; }
#else
__device__ __forceinline__ uint64_t mixi(uint64_t x) { return mix64(x); }
#endif
// record = Σ_pos mix(v_pos + (pos+1)·G) over (T, k, B_p, admitted…, B_d, #off, off…, #drop,
// drop…, #evicted, evicted…, lat) — positions as in the oracle; lanes hash in parallel.
#ifdef ASC_DL_NOINLINE  // experiments only
#define DL_ATTR __noinline__
#else
#define DL_ATTR __forceinline__  // one call site per plain kernel (log_rec in the event loop)
#endif
__device__ DL_ATTR void digest_log(Wp w, int k, int64_t T, int32_t nadm,
                                        int64_t bd, int32_t noff, int32_t ndrop, int32_t npre,
                                        int64_t lat, int32_t nch = 0) {
#if defined(ASC_DIGEST_OFF) || defined(ASC_DIGEST_OFF_LOG)  // experiments only: the checker digest's cost
  return;
#endif
  const int lane = lane_id();
  const int64_t o = ioff(k, w);
  uint64_t acc = 0;
  if (lane < 8) {
    uint64_t v, pos;
    switch (lane) {
      case 0: v = (uint64_t)T; pos = 0; break;
      case 1: v = (uint64_t)k; pos = 1; break;
      case 2: v = (uint64_t)nadm; pos = 2; break;
      case 3: v = (uint64_t)bd; pos = 3 + nadm; break;
      case 4: v = (uint64_t)noff; pos = 4 + nadm; break;
      case 5: v = (uint64_t)ndrop; pos = 5 + nadm + noff; break;
      case 6: v = (uint64_t)npre; pos = 6 + nadm + noff + ndrop; break;
      default: v = (uint64_t)lat; pos = 7 + nadm + noff + ndrop + npre; break;
    }
    acc = mixi(v + (pos + 1) * GOLD);
  }
  #pragma unroll 1
  for (int32_t j = lane; j < nadm; j += 32) acc += mixi((uint64_t)P.bp_id[o + j] + (uint64_t)(3 + j + 1) * GOLD);
  #pragma unroll 1
  for (int32_t j = lane; j < noff; j += 32)
    acc += mixi((uint64_t)P.scr_off[w.base() + j] + (uint64_t)(5 + nadm + j + 1) * GOLD);
  #pragma unroll 1
  for (int32_t j = lane; j < ndrop; j += 32)
    acc += mixi((uint64_t)P.scr_drop[w.base() + j] + (uint64_t)(6 + nadm + noff + j + 1) * GOLD);
  #pragma unroll 1
  for (int32_t j = lane; j < npre; j += 32)
    acc += mixi((uint64_t)P.scr_pre[w.base() + j] + (uint64_t)(7 + nadm + noff + ndrop + j + 1) * GOLD);
  #pragma unroll 1
  for (int32_t j = lane; j < nch; j += 32)  // Sarathi-like chunk sizes (staged in scr_off)
    acc += mixi((uint64_t)P.scr_off[w.base() + j] + (uint64_t)(8 + nadm + noff + ndrop + npre + j + 1) * GOLD);
  acc = warp_sum(acc);
  const uint64_t nr = w.SI()[k].nrec + 1;
  const uint64_t h = w.SI()[k].hash + mix64(acc + nr * GOLD2);
  __syncwarp();
  w.SI()[k].hash = h;  // uniform values, every lane stores the same words
  w.SI()[k].nrec = nr;
  __syncwarp();
}

// One formation's digest record, filled by the formation and logged by its caller: the event loop
// then holds the only digest_log call of the plain kernel.
struct DRec {
  int64_t T, bd, lat;
  int32_t nadm, noff, ndrop, npre;
  bool on;
  bool dec;  // the formation is a plain decode step, left to the caller's decode_batch
};
__device__ __forceinline__ void log_rec(Wp w, int k, const DRec& r) {
  if (r.on) digest_log(w, k, r.T, r.nadm, r.bd, r.noff, r.ndrop, r.npre, r.lat);
}

// the pure-decode record (T, k, 0, B_d, 0, 0, 0, lat): 8 lanes, 3 shuffle steps; nr = its
// formation index (1-based) on the instance
__device__ __forceinline__ uint64_t digest_decode(uint64_t h, uint64_t nr, int k, int64_t T, int64_t bd,
                                                  int64_t lat) {
#if defined(ASC_DIGEST_OFF) || defined(ASC_DIGEST_OFF_DEC)
  return h;
#endif
  const int lane = lane_id();
  const uint64_t v = lane == 0 ? (uint64_t)T : lane == 1 ? (uint64_t)k : lane == 3 ? (uint64_t)bd
                   : lane == 7 ? (uint64_t)lat : 0ull;
  const uint64_t acc = warp_sum(lane < 8 ? mixi(v + (uint64_t)(lane + 1) * GOLD) : (uint64_t)0);
  return h + mix64(acc + nr * GOLD2);
}

// ------------------------------------------------------------------------ queue helpers -------
// Every waiting queue lives in [head, head + len) of its instance region (capacity = trace size)
// and is kept sorted: LP queues by the time-invariant (key, id) of the value function (so Algorithm
// 1 reads a prefix), HP queues by id = FCFS by (arrival, id) (G26).  Admission removes a
// prefix by moving the head.
__device__ __forceinline__ int64_t qoff(const SInst& I, int k, Wp w) {
  return ioff(k, w) + I.wq_head;
}

// make room for one more entry at the tail (compacts the queue to the region start if needed)
__device__ __noinline__ void wq_compact(Wp w, int k) {
  SInst& I = w.SI()[k];
  const int lane = lane_id();
  const int64_t o = ioff(k, w);
  const int32_t h = I.wq_head, len = I.wq_len;
  #pragma unroll 1
  for (int32_t c = 0; c < len; c += 32) {
    const int32_t j = c + lane;
    int32_t xi = 0;
    int64_t xk = 0;
    if (j < len) { xi = P.wq_id[o + h + j]; xk = P.wq_key[o + h + j]; }
    __syncwarp();
    if (j < len) { P.wq_id[o + j] = xi; P.wq_key[o + j] = xk; }
    __syncwarp();
  }
  I.wq_head = 0;
  __syncwarp();
}

// insert request id in order: LP by (key, id), HP by id.  The position is searched from the tail:
// new arrivals carry the largest ids and, under the laxity key, keys near the largest.
__device__ __noinline__ void wq_insert(Wp w, int k, int32_t id) {
  SInst& I = w.SI()[k];
  const int lane = lane_id();
  if (I.wq_head + I.wq_len >= (int32_t)w.n()) wq_compact(w, k);
  const int64_t q = qoff(I, k, w);
  const int32_t len = I.wq_len;
  const int64_t key = key_of(w.base() + id, P.rq_eff[w.base() + id]);
  const bool by_id = I.hp;
  int32_t pos = len;  // number of entries ordered before the new one
  #pragma unroll 1
  for (int32_t c = len - 1; c >= 0; c -= 32) {
    const int32_t j = c - lane;
    bool after = false;  // entry j sorts after the new entry
    if (j >= 0) {
      const int32_t xi = P.wq_id[q + j];
      const int64_t xk = P.wq_key[q + j];
      after = by_id ? xi > id : (xk > key || (xk == key && xi > id));
    }
    const uint32_t m = __ballot_sync(FULL, after);
    pos -= __popc(m);
    if (m != FULL) break;  // entries are sorted: everything before this chunk sorts before
  }
  #pragma unroll 1
  for (int32_t c = len - 1; c >= pos; c -= 32) {  // shift [pos, len) up by one
    const int32_t j = c - lane;
    int32_t xi = 0;
    int64_t xk = 0;
    const bool v = j >= pos;
    if (v) { xi = P.wq_id[q + j]; xk = P.wq_key[q + j]; }
    __syncwarp();
    if (v) { P.wq_id[q + j + 1] = xi; P.wq_key[q + j + 1] = xk; }
    __syncwarp();
  }
  if (lane == 0) {
    P.wq_id[q + pos] = id;
    P.wq_key[q + pos] = key;
  }
  __syncwarp();
  I.wq_len = len + 1;
  __syncwarp();
}

// append (HP ticket: the newest arrival has the largest id, so the order is kept)
__device__ __forceinline__ void wq_append(Wp w, int k, int32_t id) {
  SInst& I = w.SI()[k];
  if (I.wq_head + I.wq_len >= (int32_t)w.n()) wq_compact(w, k);
  const int64_t q = qoff(I, k, w);
  const int32_t len = I.wq_len;
  const int64_t key = key_of(w.base() + id, P.rq_eff[w.base() + id]);
  __syncwarp();
  if (lane_id() == 0) {
    P.wq_id[q + len] = id;
    P.wq_key[q + len] = key;
  }
  I.wq_len = len + 1;
  __syncwarp();
}

// sort n request ids ascending (offload / drop lists come out in key order; the dispatch and the
// digest use id order).  Rank by counting: ids are distinct.
__device__ __noinline__ void sort_ids(Wp w, int32_t* a, int32_t n) {
  const int lane = lane_id();
  if (n <= 1) return;
  if (n <= 32) {
    int32_t x = lane < n ? a[lane] : INT32_MAX;
    const int l = lane;
#pragma unroll
    for (int kk = 2; kk <= 32; kk <<= 1)
#pragma unroll
      for (int j = kk >> 1; j > 0; j >>= 1) {
        const int32_t o = __shfl_xor_sync(FULL, x, j);
        const bool keep_min = ((l & j) == 0) == ((l & kk) == 0);
        x = keep_min ? min(x, o) : max(x, o);
      }
    __syncwarp();
    if (lane < n) a[lane] = x;
    __syncwarp();
    return;
  }
  int32_t* tmp = P.scr_tmp + w.base();
  #pragma unroll 1
  for (int32_t i = lane; i < n; i += 32) {
    const int32_t x = a[i];
    int32_t r = 0;
    #pragma unroll 1
    for (int32_t j = 0; j < n; j++) r += a[j] < x;
    tmp[r] = x;
  }
  __syncwarp();
  #pragma unroll 1
  for (int32_t i = lane; i < n; i += 32) a[i] = tmp[i];
  __syncwarp();
}

// Drop rule (G34): waiting, never prefilled, strictly past the deadline.  Stable
// compaction of the queue (order kept); dropped ids go to scr_drop in ascending id order.
__device__ __noinline__ int32_t drop_step(Wp w, int k, int64_t T) {
  SInst& I = w.SI()[k];
  const int lane = lane_id();
  const int64_t q = qoff(I, k, w);
  const int32_t len = I.wq_len;
  int32_t out = 0, nd = 0, tkd = 0;
  #pragma unroll 1
  for (int32_t c = 0; c < len; c += 32) {
    const int32_t j = c + lane;
    const bool v = j < len;
    int32_t id = 0;
    int64_t key = 0;
    bool dr = false;
    if (v) {
      id = P.wq_id[q + j];
      key = P.wq_key[q + j];
      const int64_t g = w.base() + id;
      dr = !(P.rq_fl[g] & F_EVER) && T > P.rq_dl[g];
    }
    const uint32_t mk = __ballot_sync(FULL, v && !dr), md = __ballot_sync(FULL, dr);
    if (v && !dr) { const int32_t o2 = out + __popc(mk & lanemask_lt()); P.wq_id[q + o2] = id; P.wq_key[q + o2] = key; }
    if (dr) {
      const int64_t g = w.base() + id;
      P.scr_drop[w.base() + nd + __popc(md & lanemask_lt())] = id;
      set_state(g, 2u);
      if (I.hp && (P.rq_fl[g] & F_TICK)) tkd++;
    }
    out += __popc(mk);
    nd += __popc(md);
    __syncwarp();
  }
  tkd = warp_sum(tkd);
  const int32_t tk = I.tk_live - tkd;
  __syncwarp();
  I.wq_len = out;
  I.tk_live = tk;
  __syncwarp();
  if (!I.hp && nd > 1) sort_ids(w, P.scr_drop + w.base(), nd);  // LP queue order is key order
  return nd;
}

// --------------------------------------------------------------------------- decode prep -----
// §5.4; grow each decode's KV by the blocks its next token needs (precomputed by the
// completion pass as pending bits); while short of blocks, evict the latest-arrived decode (LIFO,
// G31) by recomputation: generated tokens join its prompt, it re-enters the queue.
__device__ __forceinline__ int32_t evict(Wp w, int k) {
  SInst& I = w.SI()[k];
  const int lane = lane_id();
  int32_t np = 0;
  while (I.need_sum > I.kv_free) {
    const int32_t len = I.ds_len;
    int32_t best = -1, bslot = -1;
    #pragma unroll 1
    for (int32_t c = 0; c < len; c += 32) {
      const int32_t j = c + lane;
      if (j < len) {
        const int32_t id = slotp(w, k, j)->x;
        if (id > best) { best = id; bslot = j; }
      }
    }
    const int32_t vid = warp_max(best);
    const uint32_t who = __ballot_sync(FULL, best == vid);
    const int32_t vslot = __shfl_sync(FULL, bslot, __ffs(who) - 1);
    const int4 s = *slotp(w, k, vslot);
    const int4 last = *slotp(w, k, len - 1);
    const int64_t g = w.base() + vid;
    const int32_t kvf = I.kv_free + (s.w & HELD_MASK);  // blocks held before this step's growth
    const int32_t need = I.need_sum - (int32_t)((uint32_t)s.w >> 31);
    const int64_t cs = I.ctx_sum - s.y;
    __syncwarp();
    if (lane == 0) {
      P.rq_eff[g] = s.y;  // eff_prompt = prompt + generated = lhat
      if (P.rq_cdone) P.rq_cdone[g] = 0;
      P.rq_fl[g] += (1u << NPRE_SHIFT);
      P.scr_pre[w.base() + np] = vid;
      *slotp(w, k, vslot) = last;
    }
    I.kv_free = kvf;
    I.need_sum = need;
    I.ctx_sum = cs;
    I.ds_len = len - 1;
    __syncwarp();
    np++;
    wq_insert(w, k, vid);
  }
  return np;
}

// returns the number of evictions; leaves the growth applied (papp = 1)
__device__ __forceinline__ int32_t decode_prep(Wp w, int k) {
  SInst& I = w.SI()[k];
  if (I.papp) return 0;  // growth for the last decode step already applied
  int32_t np = 0;
  if (I.need_sum > I.kv_free) np = evict(w, k);
  const int32_t kvf = I.kv_free - I.need_sum;  // pending growth of the surviving decodes
  __syncwarp();
  I.kv_free = kvf;
  I.papp = 1;
  __syncwarp();
  return np;
}

// mark request admitted at T on instance k
__device__ __forceinline__ void admit_req(int64_t g, int k, int64_t T) {
  uint32_t f = P.rq_fl[g];
  f = (f & ~(0xffu << INST_SHIFT)) | ((uint32_t)k << INST_SHIFT) | F_EVER;
  P.rq_fl[g] = f;
  if (P.pstart[g] < 0) P.pstart[g] = T;
}

__device__ __forceinline__ void set_batch(SInst& I, int64_t T, int64_t l,
                                          int32_t bdec, int32_t nadm) {
  if (l < 0) atomicOr(P.err, ERR_RANGE);
  __syncwarp();
  I.end = T + l;
  I.batch_dec = bdec;
  I.bp_len = nadm;
  __syncwarp();
}

// ---------------------------------------------------------------- decision snapshots (diag) --
// asc_arm_snapshots: the inputs of a sampled Algorithm-1 formation (queue in (key, id) order with
// the per-entry fields asc_schedule_step takes, and the budgets) ...
__device__ __noinline__ int snap_begin(Wp w, int k, int64_t T, int64_t M, int64_t Bd, int64_t sl,
                                       int64_t Rb, int32_t len, int64_t q) {
  const SInst& I = w.SI()[k];
  if (k != P.sn_inst || w.base() != P.off[P.sn_trace]) return -1;
  const int64_t ord = (int64_t)I.nrec + 1;
  if (ord % P.sn_every != 0) return -1;
  const int64_t ns = P.sn_cnt[0], e0 = P.sn_cnt[1];
  if (ns >= P.sn_max || e0 + len > P.sn_ecap) return -1;
  const int lane = lane_id();
  for (int32_t j = lane; j < len; j += 32) {
    const int32_t id = P.wq_id[q + j];
    const int64_t g = w.base() + id;
    const uint32_t f = P.rq_fl[g];
    P.sn_ids[e0 + j] = id;
    P.sn_dl[e0 + j] = P.rq_dl[g];
    P.sn_eff[e0 + j] = P.rq_eff[g];
    P.sn_fl[e0 + j] = (uint8_t)(((f & F_EVER) ? 1u : 0u) | ((f & F_ONHP) ? 2u : 0u));
  }
  if (lane == 0) {
    int64_t* h = P.sn_hdr + 16 * ns;
    h[0] = T; h[1] = k; h[2] = P.lp_tok; h[3] = M; h[4] = Bd; h[5] = sl; h[6] = w.tbt(); h[7] = Rb;
    h[8] = len; h[9] = e0; h[14] = ord;
    P.sn_cnt[0] = ns + 1;
    P.sn_cnt[1] = e0 + len;
  }
  __syncwarp();
  return (int)ns;
}
// ... and the decision it made: admitted ids in priority order, offloaded ids ascending, latency
__device__ __noinline__ void snap_end(Wp w, int ns, int k, int32_t nadm, int32_t noff, int64_t lat) {
  const int64_t o0 = P.sn_cnt[2];
  const int lane = lane_id();
  int64_t* h = P.sn_hdr + 16 * ns;
  const bool fits = o0 + nadm + noff <= P.sn_ocap;
  if (fits) {
    const int64_t o = ioff(k, w);
    for (int32_t j = lane; j < nadm; j += 32) P.sn_out[o0 + j] = P.bp_id[o + j];
    for (int32_t j = lane; j < noff; j += 32) P.sn_out[o0 + nadm + j] = P.scr_off[w.base() + j];
  }
  __syncwarp();
  if (lane == 0) {
    h[10] = fits ? nadm : -1;  // -1: the decision did not fit out_ids
    h[11] = noff;
    h[12] = o0;
    h[13] = lat;
    if (fits) P.sn_cnt[2] = o0 + nadm + noff;
  }
  __syncwarp();
}

// --------------------------------------------------------------- LP admission (non-empty queue)
// The queue is sorted by the time-invariant (key, id), i.e. already in Algorithm 1's
// line-3 order: lines 5-13 read its prefix.  Offload (§5.3, G24) under EDF_LAXITY is the range
// key <= T + W_hp + margin right after the admitted prefix (key = deadline - prefill_us makes the
// offload test a key bound); other policies scan the whole queue.
#ifdef ASC_LA_NOINLINE  // experiments only
#define LA_ATTR __noinline__
#else
#define LA_ATTR __forceinline__
#endif
__device__ LA_ATTR int lp_admit(Wp w, int k, int64_t T, int32_t ndrop,
                                     int32_t npre, DRec& rec) {
  SInst& I = w.SI()[k];
  const int lane = lane_id();
  const int64_t o = ioff(k, w);  // running-batch list base
  const int64_t q = qoff(I, k, w);
  const int64_t Bd = I.ds_len;
  const int64_t sl = I.ctx_sum;
  // budgets (G22)
  const int64_t N = P.lp_tok, M = I.kv_free, Rb = P.lp_max - Bd;
  int64_t C = INF64, ldec = 0;
  if (Bd) {
    ldec = lat_dec_call(Bd, (int64_t)sl);
    if (ldec < 0) atomicOr(P.err, ERR_RANGE);
    C = w.tbt() - ldec;
  }
  const int32_t len = I.wq_len;
  const int snap = P.sn_hdr ? snap_begin(w, k, T, M, Bd, (int64_t)sl, Rb, len, q) : -1;
  // Algorithm 1 lines 5-13 as a strict prefix-sum scan over the sorted prefix.  Token and block
  // sums run in 32 bits: a chunk of 32 is reached only if every running sum of the previous one
  // stayed below N (< 2^25) / M (< 2^31), and a chunk adds < 2^30 (p < 2^25), so they stay < 2^32;
  // the admitted sums are below N and M.  The µs sum (prefill times up to 2^31) stays 64-bit.
  int32_t nadm = 0;
  uint64_t sp2 = 0, spc = 0;
  uint32_t sp = 0, used = 0, ct = 0, cb = 0;
  int64_t cc = 0;
  const uint32_t N32 = (uint32_t)N, M32 = (uint32_t)M;
#pragma unroll 1
  for (int r = 0; r < KPL; r++) {
    const int pos = r * 32 + lane;
    const bool valid = pos < len;
    const int32_t id = valid ? P.wq_id[q + pos] : 0;
    const int64_t g = w.base() + id;
    const int32_t p = valid ? P.rq_eff[g] : 0;
    const int64_t pf = valid ? pf_of(p) : 0;
    const uint32_t bl = valid ? (uint32_t)blk_of(p) : 0u;
    const uint32_t St = ct + warp_incl_scan((uint32_t)p);
    const uint32_t Sb = cb + warp_incl_scan(bl);
    const int64_t Sc = cc + warp_incl_scan(pf);
    const bool ok = valid && St < N32 && Sb < M32 && Sc < C && pos < Rb;
    const uint32_t m = __ballot_sync(FULL, ok);
    const int cnt = (m == FULL) ? 32 : (__ffs(~m) - 1);
    if (lane < cnt) {
      admit_req(g, k, T);
      P.bp_id[o + pos] = id;
      const uint64_t u = (uint64_t)p;
      sp += (uint32_t)p;
      sp2 += u * u;
      spc += u * ceilb(u);
      used += bl;
    }
    nadm += cnt;
    if (cnt < 32) break;
    ct = __shfl_sync(FULL, St, 31);
    cb = __shfl_sync(FULL, Sb, 31);
    cc = __shfl_sync(FULL, Sc, 31);
  }
  sp = warp_sum(sp);
  sp2 = warp_sum(sp2);
  spc = warp_sum(spc);
  used = warp_sum(used);
  // the admitted requests are the queue's prefix
  const int64_t q2 = q + nadm;
  int32_t head = I.wq_head + nadm, rem = len - nadm;
  int32_t noff = 0;
  if (w.offl() && rem > 0) {
    if (P.policy == ASC_POLICY_EDF_LAXITY && !P.look && !P.rq_koff) {
      // offload range: the prefix with key <= othr; eligible entries leave, the rest (evicted,
      // ever-prefilled requests) are packed in order at the end of the range
      const int64_t othr = T + P.W + P.margin;
      int32_t m = 0;
      #pragma unroll 1
      for (int32_t c = 0; c < rem; c += 32) {
        const int32_t j = c + lane;
        const uint32_t in = __ballot_sync(FULL, j < rem && P.wq_key[q2 + j] <= othr);
        m += __popc(in);
        if (in != FULL) break;
      }
      int32_t wpos = m;  // backward stable compaction of the kept entries inside [0, m)
      #pragma unroll 1
      for (int32_t c = m - 1; c >= 0; c -= 32) {
        const int32_t j = c - lane;
        const bool v = j >= 0;
        int32_t id = 0;
        int64_t key = 0;
        bool off = false;
        if (v) {
          id = P.wq_id[q2 + j];
          key = P.wq_key[q2 + j];
          off = !(P.rq_fl[w.base() + id] & (F_EVER | F_ONHP));
        }
        const uint32_t mk = __ballot_sync(FULL, v && !off), mo = __ballot_sync(FULL, off);
        if (v && !off) {
          const int32_t d = wpos - 1 - __popc(mk & lanemask_lt());
          P.wq_id[q2 + d] = id;
          P.wq_key[q2 + d] = key;
        }
        if (off) P.scr_off[w.base() + noff + __popc(mo & lanemask_lt())] = id;
        wpos -= __popc(mk);
        noff += __popc(mo);
        __syncwarp();
      }
      head += wpos;  // wpos = number of offloaded entries
      rem -= wpos;
    } else {
      // the whole remaining queue (in priority order); look-ahead (G50) adds the prefill time of
      // every remaining request ahead of this one
      int32_t out = 0;
      int64_t ahead = 0;
      #pragma unroll 1
      for (int32_t c = 0; c < rem; c += 32) {
        const int32_t j = c + lane;
        const bool v = j < rem;
        int32_t id = 0;
        int64_t key = 0;
        bool off = false;
        int64_t pf = 0;
        if (v) {
          id = P.wq_id[q2 + j];
          key = P.wq_key[q2 + j];
          pf = pf_of(P.rq_eff[w.base() + id]);
        }
        int64_t ex = 0;
        if (P.look) {
          const int64_t inc = warp_incl_scan(pf);
          ex = ahead + inc - pf;
          ahead += __shfl_sync(FULL, inc, 31);
        }
        if (v) {
          const int64_t g = w.base() + id;
          off = !(P.rq_fl[g] & (F_EVER | F_ONHP)) && P.rq_dl[g] - T <= pf + P.W + P.margin + ex;
        }
        const uint32_t mk = __ballot_sync(FULL, v && !off), mo = __ballot_sync(FULL, off);
        if (v && !off) {
          const int32_t d = out + __popc(mk & lanemask_lt());
          P.wq_id[q2 + d] = id;
          P.wq_key[q2 + d] = key;
        }
        if (off) P.scr_off[w.base() + noff + __popc(mo & lanemask_lt())] = id;
        out += __popc(mk);
        noff += __popc(mo);
        __syncwarp();
      }
      rem = out;
    }
    if (noff > 1) sort_ids(w, P.scr_off + w.base(), noff);  // dispatch and digest in ascending id order
  }
  const int32_t kvf = I.kv_free - (int32_t)used;
  __syncwarp();
  I.wq_head = rem > 0 ? head : 0;
  I.wq_len = rem;
  I.kv_free = kvf;
  __syncwarp();
  // dispatch offloads round-robin over the HPs, ascending id
  #pragma unroll 1
  for (int32_t j = 0; j < noff; j++) {
    const int32_t id = P.scr_off[w.base() + j];
    const int64_t g = w.base() + id;
    const int32_t rr = w.ts()->rr_hp;
    const int h = w.nlp() + rr;
    const int32_t tail = w.ts()->fl_tail;
    __syncwarp();
    if (lane == 0) {
      P.rq_fl[g] |= (F_ONHP | F_OFFL);
      w.ts()->rr_hp = (rr + 1) % w.nhp();
      if (P.delay != 0) {
        P.fl_t[w.base() + tail] = T + P.delay;
        P.fl_req[w.base() + tail] = id;
        P.fl_hp[w.base() + tail] = h;
        w.ts()->fl_tail = tail + 1;
      }
    }
    __syncwarp();
    if (P.delay == 0) wq_insert(w, h, id);
  }
  // batch (§5.4): decodes piggybacked with the admitted prefills
  const bool nonempty = nadm > 0 || Bd > 0;
  int64_t l = 0;
  if (nonempty) {
    l = nadm ? lat_batch((uint64_t)nadm, sp, sp2, spc, (uint64_t)Bd, (uint64_t)sl) : ldec;
    set_batch(I, T, l, Bd > 0, nadm);
  }
  rec = DRec{T, nonempty ? Bd : 0, l, nadm, noff, ndrop, npre, nonempty || noff || ndrop || npre};
  if (snap >= 0) snap_end(w, snap, k, nadm, noff, l);
  return nonempty ? 1 : 0;
}

// one decode-only batch of the whole decode set (LP with an empty queue, or HP) — the hot path
__device__ __forceinline__ void decode_batch(SInst& I, int k, int64_t T) {
  const int32_t bd = I.ds_len;
  const int64_t l = lat_dec_call(bd, I.ctx_sum);
  if (l < 0) atomicOr(P.err, ERR_RANGE);
  const uint64_t nr = I.nrec + 1;
  const uint64_t h = digest_decode(I.hash, nr, k, T, bd, l);
  __syncwarp();
  I.hash = h;  // uniform values: every lane stores the same words
  I.nrec = nr;
  I.end = T + l;
  I.batch_dec = 1;
  I.bp_len = 0;
  __syncwarp();
}

// returns (waiting-queue entries evaluated << 1) | (1 if a batch was formed)
__device__ __forceinline__ int64_t form_lp(Wp w, int k, int64_t T, DRec& rec) {
  SInst& I = w.SI()[k];
  int32_t ndrop = 0, npre = 0;
  if (I.wq_len == 0) {
    if (I.ds_len == 0) return 0;  // parked
    npre = decode_prep(w, k);
    if (npre == 0) {  // no eviction: the common case, a pure decode step (the caller runs it)
      rec.dec = true;
      return 1;
    }
    // the queue now holds the evicted decodes
  } else {
    ndrop = P.drop ? drop_step(w, k, T) : 0;
    npre = I.ds_len ? decode_prep(w, k) : 0;
    if (I.wq_len == 0) {
      const int64_t ev = (int64_t)I.wq_len << 1;
      const int64_t Bd = I.ds_len;
      int64_t l = 0;
      if (Bd) {
        l = lat_dec_call(Bd, I.ctx_sum);
        set_batch(I, T, l, 1, 0);
      }
      rec = DRec{T, Bd, l, 0, 0, ndrop, 0, true};  // ndrop > 0 here
      return ev | (Bd ? 1 : 0);
    }
  }
  const int64_t ev = (int64_t)I.wq_len << 1;
  return ev | lp_admit(w, k, T, ndrop, npre, rec);  // (one call site: inlined)
}

// --------------------------------------------------------------------------- HP formation ---
// FCFS prefill-first under the (elastic) token limit (G27-G28).  The
// vLLM-like baseline (G46) is the same prefill-first rule on an LP-type instance: its queue is in
// policy-key order, the limit is lp_token_budget and the batch cap applies.
__device__ __forceinline__ int32_t hp_prefill(Wp w, int k, int64_t T, uint64_t* mom) {
  SInst& I = w.SI()[k];
  const int lane = lane_id();
  const int64_t o = ioff(k, w);
  const int64_t q = qoff(I, k, w);
  int64_t limit = P.hp_tok;
  int32_t rcap = INT32_MAX;  // request cap: HPs have none
  if (!I.hp) {               // vLLM-like baseline instance (G46): N and the batch cap
    limit = P.lp_tok;
    rcap = P.lp_max - I.ds_len;
  } else if (P.elastic) {
    const int64_t mean = I.hist_cnt ? I.hist_sum / I.hist_cnt : (int64_t)P.hist_def;
    const int64_t avail = (int64_t)I.kv_free * P.bs - mean * ((int64_t)I.ds_len + 1);
    if (10 * avail > (int64_t)I.kv_total * P.bs) limit = P.hp_tok + avail;
  }
  const int32_t len = I.wq_len;
  const int64_t kvf = I.kv_free;
  int64_t ct = 0, cb = 0, used = 0;
  int32_t nadm = 0;
  uint64_t sp = 0, sp2 = 0, spc = 0;
  #pragma unroll 1
  for (int32_t c = 0; c < len; c += 32) {
    const int32_t j = c + lane;
    const bool v = j < len;
    int32_t id = 0, p = 0;
    if (v) { id = P.wq_id[q + j]; p = P.rq_eff[w.base() + id]; }
    const int64_t bl = v ? blk_of(p) : 0;
    const int64_t St = ct + warp_incl_scan((int64_t)p);
    const int64_t Sb = cb + warp_incl_scan(bl);
    const bool ok = v && j < rcap && ((j == 0 && I.hp) ? (bl <= kvf) : (St <= limit && Sb <= kvf));
    const uint32_t m = __ballot_sync(FULL, ok);
    const int cnt = (m == FULL) ? 32 : (__ffs(~m) - 1);
    if (lane < cnt) {
      admit_req(w.base() + id, k, T);
      P.bp_id[o + j] = id;
      const uint64_t u = (uint64_t)p;
      sp += u;
      sp2 += u * u;
      spc += u * ceilb(u);
      used += bl;
    }
    nadm += cnt;
    if (cnt < 32) break;
    ct = __shfl_sync(FULL, St, 31);
    cb = __shfl_sync(FULL, Sb, 31);
  }
  if (nadm == 0) return 0;
  mom[0] = warp_sum(sp);
  mom[1] = warp_sum(sp2);
  mom[2] = warp_sum(spc);
  used = warp_sum(used);
  const int32_t kvn = I.kv_free - (int32_t)used;
  const int32_t h0 = I.wq_head;  // read by every lane before any lane stores
  __syncwarp();
  I.wq_head = len > nadm ? h0 + nadm : 0;  // the admitted prefix leaves the queue
  I.wq_len = len - nadm;
  I.kv_free = kvn;
  __syncwarp();
  return nadm;
}

__device__ __forceinline__ int64_t form_hp_general(Wp w, int k, int64_t T, DRec& rec) {
  SInst& I = w.SI()[k];
  const int32_t ndrop = (P.drop && I.wq_len) ? drop_step(w, k, T) : 0;
  const int64_t ev = (int64_t)I.wq_len << 1;
  uint64_t mom[3] = {0, 0, 0};
  int32_t nadm = 0, npre = 0;
  int64_t bd = 0;
  bool batch = false;
  // prefill first; if nothing is admitted, the decodes (after eviction); if every decode was evicted
  // (G43), prefill again -- one hp_prefill call site for both attempts
  bool try_pf = I.wq_len > 0;
  #pragma unroll 1
  for (int pass = 0; pass < 2; pass++) {
    if (try_pf) {
      nadm = hp_prefill(w, k, T, mom);
      batch = nadm > 0;
    }
    if (batch || pass == 1 || I.ds_len == 0) break;
    npre = decode_prep(w, k);
    if (I.ds_len > 0) {
      batch = true;
      bd = I.ds_len;
      break;
    }
    try_pf = I.wq_len > 0;
    if (!try_pf) break;
  }
  int64_t l = 0;
  if (batch) {
    l = bd ? lat_dec_call(bd, I.ctx_sum) : lat_batch((uint64_t)nadm, mom[0], mom[1], mom[2], 0, 0);
    set_batch(I, T, l, bd > 0, bd ? 0 : nadm);
  }
  rec = DRec{T, bd, l, bd ? 0 : nadm, 0, ndrop, npre, batch || ndrop || npre};
  return ev | (batch ? 1 : 0);
}

__device__ __forceinline__ int64_t form_hp(Wp w, int k, int64_t T, DRec& rec) {
  SInst& I = w.SI()[k];
  if (I.wq_len == 0) {
    if (I.ds_len == 0) return 0;  // parked
    if (I.papp || I.need_sum <= I.kv_free) {  // decode-only batch without eviction: hot path
      decode_prep(w, k);
      rec.dec = true;  // (the caller runs it)
      return 1;
    }
  }
  return form_hp_general(w, k, T, rec);
}

// ------------------------------------------------------------- Sarathi-like baseline (G47) ---
// Decodes first (growth, LIFO preemption), then the per-batch token budget chunk_tokens - B_d is
// filled in queue order: the queue's prefix takes whole remaining prompts while their running sum
// fits; the next request gets the leftover as a partial chunk and stays at the head of the queue
// (key sentinel INT64_MIN: a partial prefill is always continued first).  Stops at the first
// request whose blocks (⌈prefilled/bs⌉, or ⌈(eff+1)/bs⌉ on the last chunk) or batch slot do not fit.
__device__ __noinline__ int64_t form_sarathi(Wp w, int k, int64_t T) {
  SInst& I = w.SI()[k];
  const int lane = lane_id();
  const int32_t ndrop = (P.drop && I.wq_len) ? drop_step(w, k, T) : 0;
  const int32_t npre = I.ds_len ? decode_prep(w, k) : 0;
  const int64_t ev = (int64_t)I.wq_len << 1;
  const int64_t o = ioff(k, w);
  const int64_t q = qoff(I, k, w);
  const int32_t Bd = I.ds_len, len = I.wq_len;
  const int64_t budget = (int64_t)P.chunk_tok - Bd, kvf = I.kv_free;
  const int32_t rcap = P.lp_max - Bd;
  const uint64_t b = P.md.b;
  int64_t crem = 0, cneed = 0;
  int32_t nfull = 0, part = 0;
  uint64_t sc = 0, aF = 0, aM = 0;
  int64_t used = 0;
  #pragma unroll 1
  for (int32_t c0 = 0; c0 < len; c0 += 32) {
    const int32_t j = c0 + lane;
    const bool v = j < len;
    int32_t id = 0, eff = 0, cd = 0;
    if (v) {
      id = P.wq_id[q + j];
      eff = P.rq_eff[w.base() + id];
      cd = P.rq_cdone[w.base() + id];
    }
    const int64_t rem = eff - cd, held = (cd + P.bs - 1) / P.bs;
    const int64_t Srem = crem + warp_incl_scan(rem);
    const int64_t Sneed = cneed + warp_incl_scan(v ? blk_of(eff) - held : (int64_t)0);
    const bool okf = v && Srem <= budget && Sneed <= kvf && j < rcap;
    const uint32_t m = __ballot_sync(FULL, okf);
    const int cnt = (m == FULL) ? 32 : (__ffs(~m) - 1);
    // the first request that is not taken whole may take the leftover budget as a partial chunk
    const int64_t left = budget - (cnt ? __shfl_sync(FULL, Srem, (cnt - 1) & 31) : crem);
    const int64_t kvl = kvf - (cnt ? __shfl_sync(FULL, Sneed, (cnt - 1) & 31) : cneed);
    int64_t c = 0, need = 0;
    bool take = false;
    if (lane < cnt) {
      c = rem;
      need = blk_of(eff) - held;
      take = true;
    } else if (lane == cnt && v && rem > left && left > 0 && j < rcap) {
      c = left;
      need = (cd + c + P.bs - 1) / P.bs - held;
      take = need <= kvl;
    }
    if (take) {
      const int64_t g = w.base() + id;
      admit_req(g, k, T);
      P.rq_cdone[g] = cd + (int32_t)c;
      P.bp_id[o + j] = id;
      P.scr_off[w.base() + j] = (int32_t)c;
      const uint64_t lc = (uint64_t)cd, cc = (uint64_t)c;
      sc += cc;
      aF += lc * cc + cc * cc;
      aM += 2 * lc + 3 * cc * ceil_div_u(lc, b) + 2 * cc + 3 * cc * ceil_div_u(cc, b);
      used += need;
    }
    nfull += cnt;
    if (cnt < 32) {
      part = __popc(__ballot_sync(FULL, take && lane == cnt));
      break;
    }
    crem = __shfl_sync(FULL, Srem, 31);
    cneed = __shfl_sync(FULL, Sneed, 31);
  }
  sc = warp_sum(sc);
  aF = warp_sum(aF);
  aM = warp_sum(aM);
  used = warp_sum(used);
  const int32_t nch = nfull + part;
  const int32_t h0 = I.wq_head;  // read by every lane before any lane stores
  __syncwarp();
  if (part && lane == 0) P.wq_key[q + nfull] = INT64_MIN;  // the partial request leads the queue
  I.wq_head = len > nfull ? h0 + nfull : 0;                  // whole prompts leave the queue
  I.wq_len = len - nfull;
  I.kv_free = (int32_t)(kvf - used);
  __syncwarp();
  const bool batch = nch > 0 || Bd > 0;
  int64_t l = 0;
  if (batch) {
    l = lat_chunked(P.md, (uint64_t)nch, sc, aF, aM, (uint64_t)Bd, (uint64_t)I.ctx_sum);
    set_batch(I, T, l, Bd > 0, nch);
  }
  if (batch || ndrop || npre) digest_log(w, k, T, nch, batch ? Bd : 0, 0, ndrop, npre, l, nch);
  return ev | (batch ? 1 : 0);
}

__device__ __forceinline__ int64_t form_sar(Wp w, int k, int64_t T) {
  SInst& I = w.SI()[k];
  if (I.wq_len == 0) {
    if (I.ds_len == 0) return 0;  // parked
    if (I.papp || I.need_sum <= I.kv_free) {  // decode-only batch without eviction: hot path
      decode_prep(w, k);
      decode_batch(I, k, T);
      return 1;
    }
  }
  return form_sarathi(w, k, T);
}

// baseline schedulers, out of line so Ascendra's event loop keeps its instruction footprint
__device__ __noinline__ int64_t form_baseline(Wp w, int k, int64_t T) {
  if (P.mode != 1) return form_sar(w, k, T);
  DRec rec;
  rec.on = false;
  rec.dec = false;
  const int64_t r = form_hp(w, k, T, rec);
  if (rec.dec) decode_batch(w.SI()[k], k, T);
  log_rec(w, k, rec);
  return r;
}

// ------------------------------------------------------------------ phase A: batch completion --
__device__ __forceinline__ void finish_req(int64_t g, int64_t T) {
  P.done[g] = T;
  set_state(g, 1u);
}

// per finished request: blocks freed, HP history, resident-ticket release (G29)
__device__ __forceinline__ void finish_sums(Wp w, int k, int64_t freed, int64_t hsum,
                                         int32_t hcnt, int32_t tkd, int64_t cfin) {
  freed = warp_sum(freed);
  hsum = warp_sum(hsum);
  hcnt = warp_sum(hcnt);
  tkd = warp_sum(tkd);
  cfin = warp_sum(cfin);
  SInst& I = w.SI()[k];
  const int32_t kvf = I.kv_free + (int32_t)freed, hc = I.hist_cnt + hcnt, tk = I.tk_live - tkd;
  const int64_t hs = I.hist_sum + hsum, cs = I.ctx_sum - cfin;
  __syncwarp();
  I.kv_free = kvf;
  I.hist_sum = hs;
  I.hist_cnt = hc;
  I.tk_live = tk;
  I.ctx_sum = cs;
  __syncwarp();
}

// prefill completions: first token, then completion or entry into the decode set
#ifdef ASC_CP_NOINLINE  // experiments only
#define CP_ATTR __noinline__
#else
#define CP_ATTR __forceinline__  // one call site (complete)
#endif
__device__ CP_ATTR void complete_prefills(Wp w, int k, int64_t T) {
  SInst& I = w.SI()[k];
  const int lane = lane_id();
  const int64_t o = ioff(k, w);
  const int32_t blen = I.bp_len;
  int32_t dlen = I.ds_len;
  int64_t freed = 0, hsum = 0, cadd = 0;
  int32_t hcnt = 0, tkd = 0;
  #pragma unroll 1
  for (int32_t c = 0; c < blen; c += 32) {
    const int32_t j = c + lane;
    const bool v = j < blen;
    bool stay = false;
    int4 s = make_int4(0, 0, 0, 0);
    if (v && P.mode == 2 && P.rq_cdone[w.base() + P.bp_id[o + j]] != P.rq_eff[w.base() + P.bp_id[o + j]]) {
      // Sarathi-like partial chunk: the request stays at the head of its queue
    } else if (v) {
      const int32_t id = P.bp_id[o + j];
      const int64_t g = w.base() + id;
      const int32_t eff = P.rq_eff[g], p = P.pl[g], out_len = P.ol[g];
      const int32_t gen = eff - p + 1;  // tokens generated after this prefill
      if (P.first[g] < 0) P.first[g] = T;
      const int32_t held = blk_of(eff);
      if (gen == out_len) {
        finish_req(g, T);
        freed += held;
        if (I.hp) { hsum += out_len; hcnt++; if (P.rq_fl[g] & F_TICK) tkd++; }
      } else {
        stay = true;
        const int32_t ctx = p + gen;
        s = make_int4(id, ctx, out_len - gen, held | (modb(ctx) << R_SHIFT));
        cadd += ctx;
      }
    }
    const uint32_t ms = __ballot_sync(FULL, stay);
    if (stay) *slotp(w, k, dlen + __popc(ms & lanemask_lt())) = s;
    dlen += __popc(ms);
  }
  freed = warp_sum(freed);
  hsum = warp_sum(hsum);
  hcnt = warp_sum(hcnt);
  tkd = warp_sum(tkd);
  cadd = warp_sum(cadd);
  const int32_t kvf = I.kv_free + (int32_t)freed, hc = I.hist_cnt + hcnt, tk = I.tk_live - tkd;
  const int64_t hs = I.hist_sum + hsum, cs = I.ctx_sum + cadd;
  __syncwarp();
  I.ds_len = dlen;
  I.kv_free = kvf;
  I.hist_sum = hs;
  I.hist_cnt = hc;
  I.tk_live = tk;
  I.ctx_sum = cs;
  __syncwarp();
}

// The decode step just executed: one pass over the slots — l̂+1, remaining−1, completions, and
// the block the next formation will need (pending bit: l̂ mod bs was 0 before the step).
__device__ __forceinline__ void complete(Wp w, int k, int64_t T) {
  SInst& I = w.SI()[k];
  const int lane = lane_id();
  if (I.batch_dec) {
    const int32_t dlen = I.ds_len;
    const int32_t bs = P.bs;
    int32_t out = 0, need = 0;
    bool anyfin = false;
    int64_t freed = 0, hsum = 0, cfin = 0;
    int32_t hcnt = 0, tkd = 0;
    #pragma unroll 1
    for (int32_t c = 0; c < dlen; c += 32) {
      const int32_t j = c + lane;
      const bool v = j < dlen;
      int4 s = make_int4(0, 0, 1, 0);
      if (v) s = *slotp(w, k, j);
      const int32_t held = (s.w & HELD_MASK) + (int32_t)((uint32_t)s.w >> 31);  // growth applied
      const int32_t r = (s.w >> R_SHIFT) & 0x1ff;
      const bool pend = r == 0;
      const int32_t r2 = r + 1 == bs ? 0 : r + 1;
      s.y += 1;
      s.z -= 1;
      s.w = held | (r2 << R_SHIFT) | (pend ? PEND : 0);
      const bool fin = v && s.z == 0;
      const uint32_t mf = __ballot_sync(FULL, fin);
      const uint32_t mk = __ballot_sync(FULL, v && !fin);
      need += __popc(__ballot_sync(FULL, v && !fin && pend));
      // stable compaction (positions == j until the first completion): every lane's read is
      // ordered before the in-place writes
      __syncwarp();
      if (v && !fin) *slotp(w, k, out + __popc(mk & lanemask_lt())) = s;
      if (mf) {
        anyfin = true;
        if (fin) {
          const int64_t g = w.base() + s.x;
          finish_req(g, T);
          freed += held;
          cfin += s.y;
          if (I.hp) { hsum += P.ol[g]; hcnt++; if (P.rq_fl[g] & F_TICK) tkd++; }
        }
      }
      out += __popc(mk);
    }
    const int64_t cs = I.ctx_sum + dlen;  // every decode gained one token of context
    __syncwarp();
    I.ctx_sum = cs;
    I.ds_len = out;
    I.need_sum = need;
    I.papp = 0;
    __syncwarp();
    if (anyfin) finish_sums(w, k, freed, hsum, hcnt, tkd, cfin);
  }
  if (I.bp_len) complete_prefills(w, k, T);
  __syncwarp();
  I.bp_len = 0;
  I.batch_dec = 0;
  I.end = INF64;
  __syncwarp();
}

// --------------------------------------------------------------------- controller routing ---
template <bool PLAIN>
__device__ __forceinline__ void route(Wp w, int32_t id) {
  const int n_lp = PLAIN ? P.n_lp : w.nlp(), K = PLAIN ? P.K : w.K();
  if (PLAIN ? (P.tickets && P.n_hp >= 1) : w.tickets()) {
    #pragma unroll 1
    for (int h = n_lp; h < K; h++) {
      if (w.SI()[h].ticket) {
        const int32_t tk = w.SI()[h].tk_live + 1;
        __syncwarp();
        if (lane_id() == 0) P.rq_fl[w.base() + id] |= (F_TICK | F_ONHP);
        w.SI()[h].ticket = 0;
        w.SI()[h].tk_live = tk;
        __syncwarp();
        wq_append(w, h, id);  // the newest arrival has the largest id: stays sorted
        return;
      }
    }
  }
  const int32_t rr = w.ts()->rr_lp;
  wq_insert(w, rr, id);
  w.ts()->rr_lp = (rr + 1) == n_lp ? 0 : rr + 1;
  __syncwarp();
}

__device__ __noinline__ void deliver(Wp w, int64_t T) {
  while (w.ts()->fl_head < w.ts()->fl_tail && P.fl_t[w.base() + w.ts()->fl_head] == T) {
    const int32_t head = w.ts()->fl_head;
    const int32_t id = P.fl_req[w.base() + head];
    const int h = P.fl_hp[w.base() + head];
    wq_insert(w, h, id);
    w.ts()->fl_head = head + 1;
    __syncwarp();
  }
}

// ---------------------------------------------------------------------- phase F: decode runs --
// Between external events (the next arrival; for an HP also any LP formation that could offload
// and any in-flight delivery) an instance whose queue is empty and whose running batch is a pure
// decode batch evolves on its own: its next steps are decode-only batches of the same B_d
// requests until the first completion (event min(rem) - 1) or the first step whose block growth
// would not fit (eviction).  Those steps are evaluated 32 at a time, one per lane: block growth
// from a histogram of l̂ mod bs, Σl̂ in closed form, latencies in parallel (Eq. 4-5), start times by
// a prefix sum, and the per-instance digest chain applied in order.  Exactly the same formations,
// times and digest as stepping them one by one through the event loop.
#ifdef ASC_RD_NOINLINE  // experiments only
#define RD_ATTR __noinline__
#else
#define RD_ATTR __forceinline__  // one call site (phase F): no call, no callee-saved register traffic
#endif
__device__ RD_ATTR int64_t run_decode(Wp w, int k, int64_t T_limit) {
  SInst& I = w.SI()[k];
  const int lane = lane_id();
  const int32_t bs = P.bs;
  if (I.ds_len == 0 || bs > 128 || !I.papp) return 0;
  const bool hp = I.hp;
  // two histograms of l̂ mod bs (current slots / survivors of the next completion), plus the
  // histogram of the slots that would finish at the next completion event
  int32_t* hA = reinterpret_cast<int32_t*>(w.buf());  // w.buf() holds 256 ints: two histograms
  int32_t* hB = hA + 128;
  int32_t Bd = I.ds_len;
  int64_t E = I.end, S = I.ctx_sum;
  int32_t kvf = I.kv_free;
  uint64_t h = I.hash, nr = I.nrec;
  int64_t total = 0;
  int64_t hsum_all = 0;
  int32_t hcnt_all = 0, tkd_all = 0;
  // pass A: histogram + minimum remaining tokens of the current slots
  #pragma unroll 1
  for (int i = lane; i < 128; i += 32) hA[i] = 0;
  __syncwarp();
  int32_t mrem = INT32_MAX;
  #pragma unroll 1
  for (int32_t c = 0; c < Bd; c += 32) {
    const int32_t j = c + lane;
    if (j < Bd) {
      const int4 sl = *slotp(w, k, j);
      mrem = min(mrem, sl.z);
      atomicAdd(&hA[(sl.w >> R_SHIFT) & 0x1ff], 1);
    }
  }
  mrem = warp_min(mrem);
  __syncwarp();
  while (true) {
    const uint64_t cpart = mixi((uint64_t)k + 2 * GOLD) + mixi(3 * GOLD) + mixi((uint64_t)Bd + 4 * GOLD) +
                           mixi(5 * GOLD) + mixi(6 * GOLD) + mixi(7 * GOLD);
    const int32_t Jmax = mrem - 1;  // decode-only events before the next completion
    int32_t J = 0;
    int64_t tcarry = 0, ncarry = 0;
    // ---- lane-parallel segment: events c = 0 .. Jmax-1 (no completion among them)
    while (J < Jmax) {
      const int32_t c = J + lane;
      const int32_t cm = modb(c);
      const int32_t need = hA[cm == 0 ? 0 : bs - cm];  // slots with (r0 + c) mod bs == 0
      const int64_t cum = ncarry + warp_incl_scan(need);
      // (the fp64 evaluation inlined here: one lane per decode event, the hottest latency site)
      const int64_t lc = lat_decode<true>(P.md, (uint64_t)Bd, (uint64_t)(S + (int64_t)(c + 1) * Bd));
      const int64_t incl = warp_incl_scan(lc < 0 ? (int64_t)0 : lc);
      const int64_t tc = E + tcarry + incl - (lc < 0 ? 0 : lc);  // formation time of event c
      const bool ok = c < Jmax && tc < T_limit && cum <= kvf && lc > 0;
      const uint32_t m = __ballot_sync(FULL, ok);
      const int n = (m == FULL) ? 32 : (__ffs(~m) - 1);
      const uint64_t rec = cpart + mixi((uint64_t)tc + GOLD) + mixi((uint64_t)lc + 8 * GOLD);
#if !defined(ASC_DIGEST_OFF) && !defined(ASC_DIGEST_OFF_DEC)
      h += warp_sum(lane < n ? mix64(rec + (nr + (uint64_t)c + 1) * GOLD2) : 0ull);
#endif
      if (n > 0) {
        ncarry = __shfl_sync(FULL, cum, n - 1);
        tcarry = __shfl_sync(FULL, incl, n - 1) + tcarry;
      }
      J += n;
      if (n < 32) break;
    }
    const int64_t Et = E + tcarry;  // time of event J (a completion event iff J == Jmax)
    // ---- can event J (the completion) be processed here?  Conservative KV check from the
    // histogram (finishing slots included): the main loop handles it if eviction might be needed
    const int32_t cJ = modb(J);
    const int64_t needJ = hA[cJ == 0 ? 0 : bs - cJ];
    const bool doC = J == Jmax && Et < T_limit && needJ <= kvf - ncarry;
    const int32_t nstep = J + (doC ? 1 : 0);
    if (nstep == 0) break;
    // ---- pass B: apply the J decode steps (and the completion event J when doC)
    #pragma unroll 1
    for (int i = lane; i < 128; i += 32) hB[i] = 0;
    __syncwarp();
    int32_t out = 0, mrem2 = INT32_MAX, need2 = 0;
    int64_t freed = 0, hsum = 0, csum = 0;
    int32_t hcnt = 0, tkd = 0;
    #pragma unroll 1
    for (int32_t c0 = 0; c0 < Bd; c0 += 32) {
      const int32_t j = c0 + lane;
      const bool v = j < Bd;
      int4 sl = make_int4(0, 0, 1 << 30, 0);
      if (v) sl = *slotp(w, k, j);
      const int32_t r0 = (sl.w >> R_SHIFT) & 0x1ff;
      const int32_t pend0 = (int32_t)((uint32_t)sl.w >> 31);
      // growth applied at formations 0 .. nstep-1 uses the pending bits of completions 0 .. nstep-1
      // held after nstep completions = held_base + pend0 + #{c in [0, nstep-2] : (r0 + c) % bs == 0}
      const int32_t first = r0 == 0 ? 0 : bs - r0;
      const int32_t last = nstep - 2;
      const int32_t grown = last >= first ? 1 + divb(last - first) : 0;
      const int32_t held = (sl.w & HELD_MASK) + pend0 + grown;
      const int32_t rN = modb(r0 + nstep);
      const bool pend = nstep > 0 && modb(r0 + nstep - 1) == 0;
      sl.y += nstep;
      sl.z -= nstep;
      sl.w = held | (rN << R_SHIFT) | (pend ? PEND : 0);
      const bool fin = v && doC && sl.z == 0;
      const bool keep = v && !fin;
      const uint32_t mk = __ballot_sync(FULL, keep);
      __syncwarp();  // every lane's slot read is ordered before the in-place compaction below
      if (keep) {
        *slotp(w, k, out + __popc(mk & lanemask_lt())) = sl;
        mrem2 = min(mrem2, sl.z);
        atomicAdd(&hB[rN], 1);
        need2 += pend ? 1 : 0;
        csum += sl.y;
      }
      if (fin) {  // completion at Et: done, KV freed, HP history / ticket bookkeeping
        const int64_t g = w.base() + sl.x;
        finish_req(g, Et);
        freed += held;  // held_base after nstep completions = blocks held when it finishes
        if (hp) { hsum += P.ol[g]; hcnt++; if (P.rq_fl[g] & F_TICK) tkd++; }
      }
      out += __popc(mk);
    }
    mrem2 = warp_min(mrem2);
    need2 = warp_sum(need2);
    csum = warp_sum(csum);
    if (doC) {
      freed = warp_sum(freed);
      hsum = warp_sum(hsum);
      hcnt = warp_sum(hcnt);
      tkd = warp_sum(tkd);
    }
    __syncwarp();
    total += J;
    kvf -= (int32_t)ncarry;
    nr += (uint64_t)J;
    if (!doC) {  // the run ends before event J: event J (at Et) is left to the event loop
      E = Et;
      S = csum;
      break;
    }
    // ---- the formation at Et after the completion: a decode-only batch of the survivors
    kvf += (int32_t)freed;
    hsum_all += hsum;
    hcnt_all += hcnt;
    tkd_all += tkd;
    Bd = out;
    S = csum;
    if (Bd == 0) {  // everything finished: the instance parks
      E = INF64;
      break;
    }
    kvf -= need2;  // growth for the survivors' next token (fits: needJ <= kvf - ncarry above)
    const int64_t l = lat_dec_call(Bd, S);
    if (l < 0) atomicOr(P.err, ERR_RANGE);
    nr += 1;
    h = digest_decode(h, nr, k, Et, Bd, l);
    total += 1;
    E = Et + l;
    // the survivors become the current slots (their pending bits were just applied: papp = 1)
    int32_t* t = hA; hA = hB; hB = t;
    mrem = mrem2;
    if (E >= T_limit) break;
  }
  if (total == 0) return 0;
  const int64_t hs = I.hist_sum + hsum_all;
  const int32_t hc = I.hist_cnt + hcnt_all, tk = I.tk_live - tkd_all;
  const bool issue = hp && w.tickets() && !I.ticket && I.wq_len == 0 && tk == 0;  // phase E
  __syncwarp();
  I.kv_free = kvf;
  I.ctx_sum = S;
  I.end = E;
  I.hash = h;
  I.nrec = nr;
  I.ds_len = Bd;
  I.papp = 1;
  I.hist_sum = hs;
  I.hist_cnt = hc;
  I.tk_live = tk;
  if (Bd == 0) { I.batch_dec = 0; I.bp_len = 0; }
  if (issue) I.ticket = 1;
  __syncwarp();
  return total;
}

__device__ __noinline__ void init_trace(Wp w, int trace) {
  const int lane = lane_id();
  if (lane == 0) { w.ts()->rr_lp = w.ts()->rr_hp = w.ts()->fl_head = w.ts()->fl_tail = 0; }
  const int64_t ttft = P.ttft[trace];
  #pragma unroll 1
  for (int64_t i = lane; i < w.n(); i += 32) {
    const int64_t g = w.base() + i;
    P.rq_dl[g] = P.arr[g] + (P.rttft ? P.rttft[g] : ttft);
    P.rq_eff[g] = P.pl[g];
    if (P.rq_cdone) P.rq_cdone[g] = 0;
    P.rq_fl[g] = 0xffu << INST_SHIFT;
    P.first[g] = -1;
    P.done[g] = -1;
    P.pstart[g] = -1;
  }
  if (lane < w.K()) {
    SInst& I = w.SI()[lane];
    I.hp = lane >= w.nlp();
    I.kv_total = I.kv_free = I.hp ? P.kv_hp : P.kv_lp;
    I.end = INF64; I.hist_sum = 0; I.ctx_sum = 0; I.hash = 0; I.nrec = 0; I.wq_head = 0;
    I.wq_len = I.ds_len = I.bp_len = I.hist_cnt = I.need_sum = 0;
    I.batch_dec = I.tk_live = 0;
    I.papp = 1;
    I.ticket = (I.hp && w.tickets()) ? 1 : 0;  // issued at t = 0 (G29)
  }
  __syncwarp();
}

__device__ __noinline__ void finish_trace(Wp w, int trace, int64_t decisions,
                                          int64_t evals) {
  const int lane = lane_id();
  bool stuck = false;
  if (lane < w.K()) stuck = w.SI()[lane].wq_len > 0 || w.SI()[lane].ds_len > 0;
  if (__any_sync(FULL, stuck) && lane == 0) atomicOr(P.err, ERR_INVARIANT);
  #pragma unroll 1
  for (int64_t i = lane; i < w.n(); i += 32) {
    const int64_t g = w.base() + i;
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
    #pragma unroll 1
    for (int k = 0; k < w.K(); k++) d = mix64(d ^ w.SI()[k].hash);
    P.digest[trace] = d;
    if (P.decisions) P.decisions[trace] = decisions;
#ifdef ASC_DEBUG_CLOCK  // experiments only: per-trace finish time (ns) in place of evaluations
    {  // finish time (ns, low 48 bits) and the SM the trace ran on (bits 48-63)
      uint64_t tns;
      uint32_t smid;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tns));
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      evals = (int64_t)(((uint64_t)smid << 48) | (tns & ((1ull << 48) - 1)));
    }
#endif
    if (P.evals) P.evals[trace] = evals;
  }
  __syncwarp();
}

// minimum over the lanes < K (<= 16) of a warp, lanes >= K holding INF64; returned to every lane
// minimum over the warp (lanes past the instances hold INF64): the high words by one REDUX, then the
// low words of the lanes holding that high word by another
__device__ __forceinline__ int64_t kmin64(int64_t v, int K) {
  const int32_t hi = (int32_t)(v >> 32);
  const int32_t mh = __reduce_min_sync(FULL, hi);
  const uint32_t ml = __reduce_min_sync(FULL, hi == mh ? (uint32_t)v : 0xffffffffu);
  return (int64_t)(((uint64_t)(uint32_t)mh << 32) | ml);
}

// MINB = CTAs per SM the register budget must allow (8 -> 64 registers/thread ... 4 -> 128).  The
// launch picks the largest budget that still keeps every trace of the call resident at once
// (T <= SMs x MINB x SW): a trace is a serial chain, so registers beat extra resident warps
// only while no trace waits for a slot.
// PLAIN: Ascendra with the ctx's topology for every trace (the common case): topology, tickets
// and the scheduler come from the constant bank, so none of them is live across the event loop's
// out-of-line calls.
template <int MINB, bool PLAIN>
__global__ void __launch_bounds__(SW * 32, MINB) sim_kernel() {
  const int lane = threadIdx.x & 31;
  Wp w;
  while (true) {
    int trace = 0;
    if (lane == 0) trace = atomicAdd(P.next_trace, 1);
    trace = __shfl_sync(FULL, trace, 0);
    if (trace >= P.T) break;
    if (lane == 0) {
      TS* t = w.ts();
      const int64_t b = P.off[trace];
      t->base = b;
      t->n = P.off[trace + 1] - b;
      t->tbt = P.tbt[trace];
      t->n_lp = P.tr_nlp ? P.tr_nlp[trace] : P.n_lp;
      t->n_hp = P.tr_nhp ? P.tr_nhp[trace] : P.n_hp;
      t->K = t->n_lp + t->n_hp;
      t->sw = (P.offl && t->n_hp >= 1 ? 1 : 0) | (P.tickets && t->n_hp >= 1 ? 2 : 0);
    }
    __syncwarp();
    const int K = PLAIN ? P.K : w.K(), n_lp = PLAIN ? P.n_lp : w.nlp();
    init_trace(w, trace);
    int64_t next = 0, next_arr = w.n() > 0 ? P.arr[w.base()] : INF64, decisions = 0, evals = 0;
    // Lane k < K mirrors instance k in the checks below (one shared-memory load per lane, minima
    // by shuffles, instance sets by ballots), instead of serial loops over the instances.  Every
    // phase only changes the instance it processes, so taking each set before the phase visits it
    // in ascending instance order is the canonical A-E order of DESIGN.md §2.
    const bool inst = lane < K;
    while (true) {
      const int64_t e = inst ? w.SI()[lane].end : INF64;
      int64_t T = kmin64(e, K);
      T = next_arr < T ? next_arr : T;
      const bool flight = w.ts()->fl_head < w.ts()->fl_tail;
      if (flight) {
        const int64_t tf = P.fl_t[w.base() + w.ts()->fl_head];
        T = tf < T ? tf : T;
      }
      if (T == INF64) break;
      // A. completions in instance order
      for (uint32_t m = __ballot_sync(FULL, inst && e == T); m; m &= m - 1) complete(w, __ffs(m) - 1, T);
      // B. offload deliveries (FIFO = time order)
      if (flight) deliver(w, T);
      // C. arrivals, ascending id
      while (next_arr == T) {
        route<PLAIN>(w, (int32_t)next);
        next++;
        next_arr = next < w.n() ? P.arr[w.base() + next] : INF64;
      }
      // D. formations of idle instances, LPs (lower indices) before HPs
      for (uint32_t m = __ballot_sync(FULL, inst && w.SI()[lane].end == INF64); m; m &= m - 1) {
        const int k = __ffs(m) - 1;
        DRec rec;
        rec.on = false;
        rec.dec = false;
        const int64_t r = k >= n_lp ? form_hp(w, k, T, rec)
                                    : ((PLAIN || P.mode == 0) ? form_lp(w, k, T, rec) : form_baseline(w, k, T));
        if (rec.dec) decode_batch(w.SI()[k], k, T);  // one site for both instance kinds
        log_rec(w, k, rec);
        decisions += r & 1;
        evals += r >> 1;
      }
      // E. tickets (G29)
      if (PLAIN ? (P.tickets && P.n_hp >= 1) : w.tickets()) {
        if (lane >= n_lp && lane < K) {
          SInst& I = w.SI()[lane];
          if (!I.ticket && I.wq_len == 0 && I.tk_live == 0) I.ticket = 1;
        }
        __syncwarp();
      }
      // F. decode runs of independent instances up to their next possible interaction: an LP until
      // the next arrival; an HP also until any LP formation that could offload, or a delivery
      int64_t ef = INF64;
      int32_t wl = 0, bd = 0, bp = 0;
      if (inst) {
        const SInst& I = w.SI()[lane];
        ef = I.end;
        wl = I.wq_len;
        bd = I.batch_dec;
        bp = I.bp_len;
      }
      int64_t tl_hp = kmin64(lane < n_lp && wl > 0 ? ef : INF64, K);
      tl_hp = next_arr < tl_hp ? next_arr : tl_hp;
      if (w.ts()->fl_head < w.ts()->fl_tail) {
        const int64_t tf = P.fl_t[w.base() + w.ts()->fl_head];
        tl_hp = tf < tl_hp ? tf : tl_hp;
      }
      // LP k only receives arrivals: round-robin from rr_lp (an arrival taken by an HP's ticket
      // does not advance it), so none reaches k before the ((k - rr_lp) mod n_lp)-th upcoming one
      int64_t lim = tl_hp;
      if (lane < n_lp) {
        const int32_t rr = w.ts()->rr_lp;
        const int64_t j = next + (lane >= rr ? lane - rr : lane - rr + n_lp);
        lim = j < w.n() ? P.arr[w.base() + j] : INF64;
      }
      for (uint32_t m = __ballot_sync(FULL, inst && ef < lim && bd && bp == 0 && wl == 0); m; m &= m - 1) {
        const int k = __ffs(m) - 1;
        decisions += run_decode(w, k, __shfl_sync(FULL, lim, k));
      }
    }
    finish_trace(w, trace, decisions, evals);
  }
}

// per-warp shared-memory layout: top-K buffer, decode slots, instance states, controller state
size_t sim_smem_per_warp(int K, int32_t* o_sd = nullptr, int32_t* o_si = nullptr, int32_t* o_ts = nullptr) {
  const size_t sd = 64 * sizeof(KI), si = sd + (size_t)K * DCAP * sizeof(int4);
  const size_t ts = si + (size_t)K * sizeof(SInst);
  if (o_sd) { *o_sd = (int32_t)sd; *o_si = (int32_t)si; *o_ts = (int32_t)ts; }
  return (ts + sizeof(TS) + 15) & ~size_t(15);
}

// liveness / layout validation (ASC_E_CONFIG / ASC_E_INVAL before simulating)
__global__ void validate_traces(int64_t R) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && P.off[P.T] != R) atomicOr(P.err, ERR_INVAL);
  #pragma unroll 1
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < P.T; t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t nl = P.tr_nlp ? P.tr_nlp[t] : P.n_lp, nh = P.tr_nhp ? P.tr_nhp[t] : P.n_hp;
    if (nl < 1 || nh < 0 || nl + nh > P.K || (P.mode != 0 && nh != 0)) atomicOr(P.err, 8);
  }
  #pragma unroll 1
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
  #pragma unroll 1
  for (int t = w; t < T; t += nw) {
    const int64_t lo = off[t], hi = off[t + 1];
    const int64_t tt = ttft[t], tb = tbt[t];
    uint64_t g = 0;
    // GU requests per lane per pass, every field loaded before any test (branch-free streaming:
    // the loads of a pass are independent, so several are in flight per warp)
    constexpr int GU = 4;
    #pragma unroll 1
    for (int64_t i0 = lo + lane; i0 < hi; i0 += 32 * GU) {
      uint32_t st[GU];
      int64_t f[GU], a[GU], d[GU], sl[GU];
      int32_t o[GU];
      #pragma unroll
      for (int u = 0; u < GU; u++) {
        const int64_t i = i0 + 32 * u;
        const bool v = i < hi;
        st[u] = v ? __ldcs(status + i) : 0u;
        f[u] = v ? __ldcs(first + i) : 0;
        a[u] = v ? __ldcs(arr + i) : 0;
        o[u] = v ? __ldcs(ol + i) : 1;
        d[u] = v ? __ldcs(done + i) : 0;
        sl[u] = (v && rttft) ? __ldcs(rttft + i) : tt;
      }
      #pragma unroll
      for (int u = 0; u < GU; u++) {
        // P:451 / G35: completed, TTFT within the SLO, mean TBT within the SLO (out = 1: no TBT)
        const bool ok = (st[u] & 3u) == 1u && f[u] - a[u] <= sl[u] &&
                        (o[u] <= 1 || d[u] - f[u] <= tb * (int64_t)(o[u] - 1));
        g += ok ? 1u : 0u;
      }
    }
    g = warp_sum(g);
    if (lane == 0) {
      good[t] = g;
      total[t] = (uint64_t)(hi - lo);
      if (hi == lo) atomicOr(err, 16);
    }
  }
}

cudaError_t upload_params(const SimP& h, cudaStream_t s) {
  return cudaMemcpyToSymbolAsync(P, &h, sizeof(SimP), 0, cudaMemcpyHostToDevice, s);
}

// the constant-bank parameters are per device: simulate calls on one device are serialised
std::mutex g_sim_mu[64];

}  // namespace

namespace asc {

asc_status launch_simulate(asc_ctx* c, const asc_traces* tr, asc_outcomes* out, int64_t R) {
  const asc_config& cf = c->cfg;
  const int K = cf.topo.n_lp + cf.topo.n_hp;
  const int32_t T = tr->T;
  size_t need = (size_t)R * (8 + 4 + 4) + (size_t)K * R * (8 + 4 + 16 + 4) + (size_t)R * 16 +
                (cf.flags.offload_delay_us ? (size_t)R * 16 : 0) +
                (cf.flags.scheduler == 2 ? (size_t)R * 4 : 0) + 64 * 1024;
  asc_status st = ensure_ws(c, need);
  if (st) return st;
  Arena ar{c->ws, c->ws_cap};
  SimP P;
  P.md = c->md;
  P.pf_tab = c->d_pf_tab;
  P.pt = c->pt_size;
  P.n_lp = cf.topo.n_lp; P.n_hp = cf.topo.n_hp; P.K = K; P.bs = cf.topo.block_tokens;
  P.bs_m = ((uint64_t(1) << 38) + (uint64_t)P.bs - 1) / (uint64_t)P.bs;
  P.ab_m = ((uint64_t(1) << 38) + c->md.b - 1) / c->md.b;
  P.ab_fast = c->md.b <= 4096 ? 1 : 0;
  P.lp_max = cf.topo.lp_max_batch; P.lp_tok = cf.topo.lp_token_budget; P.hp_tok = cf.topo.hp_token_budget;
  P.policy = cf.flags.policy;
  P.offl = cf.flags.offload ? 1 : 0;    // per trace: and n_hp >= 1
  P.tickets = cf.flags.tickets ? 1 : 0;
  P.tr_nlp = tr->n_lp;
  P.tr_nhp = tr->n_hp;
  P.look = cf.flags.offload_rule;
  P.kw0 = cf.flags.key_w[0]; P.kw1 = cf.flags.key_w[1]; P.kw2 = cf.flags.key_w[2];
  P.rq_koff = tr->req_key_offset_us;
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
  P.ds_g = ar.take<int4>((size_t)K * R);
  P.bp_id = ar.take<int32_t>((size_t)K * R);
  P.scr_drop = ar.take<int32_t>(R);
  P.scr_pre = ar.take<int32_t>(R);
  P.scr_off = ar.take<int32_t>(R);
  P.scr_tmp = ar.take<int32_t>(R);
  if (cf.flags.offload_delay_us) {
    P.fl_t = ar.take<int64_t>(R);
    P.fl_req = ar.take<int32_t>(R);
    P.fl_hp = ar.take<int32_t>(R);
  } else {
    P.fl_t = nullptr; P.fl_req = nullptr; P.fl_hp = nullptr;
  }
  P.next_trace = ar.take<int>(1);
  P.err = c->d_err;
  P.sn_hdr = nullptr;
  if (c->snap_armed) {  // consumed by this call
    const asc_snapshots& sn = c->snap;
    P.sn_hdr = sn.hdr; P.sn_cnt = sn.counts; P.sn_ids = sn.ids; P.sn_dl = sn.deadline_us;
    P.sn_eff = sn.eff_prompt; P.sn_fl = sn.flags; P.sn_out = sn.out_ids;
    P.sn_trace = sn.trace; P.sn_inst = sn.instance; P.sn_max = sn.max_snaps;
    P.sn_every = sn.every; P.sn_ecap = sn.entry_cap; P.sn_ocap = sn.out_cap;
    cudaMemsetAsync(sn.counts, 0, 3 * sizeof(int64_t), c->stream);
    if (sn.trace >= T) P.sn_hdr = nullptr;
    c->snap_armed = false;
  }
  P.pw = (int32_t)sim_smem_per_warp(K, &P.o_sd, &P.o_si, &P.o_ts);
  P.mode = cf.flags.scheduler;
  P.chunk_tok = cf.flags.chunk_tokens;
  P.rq_cdone = P.mode == 2 ? ar.take<int32_t>(R) : nullptr;
  cudaStream_t sm = c->stream;
  std::lock_guard<std::mutex> lock(g_sim_mu[c->device & 63]);
  cudaError_t ue = upload_params(P, sm);
  if (ue != cudaSuccess) return cuda_check(c, ue, "simulate parameters");
  int64_t launches = 0;
  if (R > 0 || T > 0) {
    const int64_t n = R > T ? R : T;
    const int64_t gb = (n + 255) / 256;
    validate_traces<<<(unsigned)(gb < 4096 ? gb : 4096), 256, 0, sm>>>(R);
    launches++;
    asc_status v = collect_errors(c, "simulate_batch validation");
    if (v) return v;
  }
  cudaMemsetAsync(P.next_trace, 0, sizeof(int), sm);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  const size_t smem = SW * sim_smem_per_warp(K);
  // register budget: fewest resident CTAs per SM that still hold every trace (min 4), and never
  // more than shared memory allows (1 KB per CTA is reserved by the runtime)
  int smem_sm = 228 * 1024;
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, c->device);
  int minb = (int)(smem_sm / (smem + 1024));
  minb = minb > 8 ? 8 : minb;
  if (minb < 1) return fail(c, ASC_E_CONFIG, "simulate: per-CTA shared memory exceeds the SM");
  for (int m = 4; m < minb; m++)
    if ((int64_t)T <= (int64_t)sms * m * SW) { minb = m; break; }
  if (minb < 4) minb = 4;  // (K so large that fewer than 4 CTAs fit: the launch itself reports it)
  if (const char* f = getenv("ASC_SIM_MINB")) {  // experiments only: force the register budget
    const int m = atoi(f);
    if (m >= 4 && m <= 8) minb = m;
  }
  const bool plain = P.mode == 0 && !tr->n_lp && !tr->n_hp;
  void (*const tab[2][5])() = {
      {sim_kernel<4, false>, sim_kernel<5, false>, sim_kernel<6, false>, sim_kernel<7, false>, sim_kernel<8, false>},
      {sim_kernel<4, true>, sim_kernel<5, true>, sim_kernel<6, true>, sim_kernel<7, true>, sim_kernel<8, true>}};
  void (*kern)() = tab[plain ? 1 : 0][minb - 4];
  int64_t blocks = ((int64_t)T + SW - 1) / SW;
  const int64_t cap = (int64_t)sms * minb;
  if (blocks > cap) blocks = cap;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_check(c, e, "simulate smem attribute");
  }
  if (blocks > 0) {
    cudaEventRecord(c->ev0, sm);
    kern<<<(unsigned)blocks, SW * 32, smem, sm>>>();
    cudaEventRecord(c->ev1, sm);
    c->timed = true;
    launches++;
  }
  c->last_kernel_launches = launches;
  cudaError_t le = cudaGetLastError();
  if (le == cudaSuccess) le = cudaStreamSynchronize(sm);  // the parameters stay in use until here
  return cuda_check(c, le, "simulate launch");
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
