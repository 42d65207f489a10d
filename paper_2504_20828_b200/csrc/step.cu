// step.cu — asc_schedule_step: the stateless LP decision over S segments.
//
// Design:
//   plan   : per segment, #warp-tasks = max(1, ceil(Q_s / 16384)); exclusive scans give each
//            segment its first task and (for segments of > 1 task) its first candidate slot, and
//            a task -> segment map.
//   k1     : one warp per task streams its <= 16384 entries once: each lane owns 4 consecutive
//            entries per 128-entry group (128-bit loads of deadline/eff_prompt, 32-bit flags),
//            evaluates a1 (prefill latency via the ctx's device table), the key (a2, branch-free),
//            the drop and offload predicates (a5, as ballot bitmasks) and keeps the smallest
//            (key, pos) entries Algorithm 1 could admit in a register-resident bitonic list (a3).
//            Single-task segments finish in place: Algorithm 1 prefix scan (a4), batch latency
//            (a6), admitted bits removed from the offload mask, popc/scan compaction (a5).
//   k2     : one CTA per multi-task segment merges the per-task lists (bitonic, warp shuffles
//            + shared-memory tree), runs Algorithm 1, clears admitted bits, scans task counts.
//   k3     : one warp per multi-task task expands its masks into id-ascending output indices.
// HBM traffic per entry: 13 B read (+4 B prefill_us if requested) + 4 B per output index;
// multi-task segments add 0.25 B/entry of mask traffic and 1.5 KB per task of candidates.
#include <mutex>
#include <type_traits>

#include "asc_internal.h"

using namespace asc;

namespace {

constexpr int KPL = 4;             // K = 128 = ASC_MAX_BATCH
constexpr int CH = 16384;          // entries per warp task
constexpr int GE = 128;            // entries per warp iteration (lane l: entries l, 32+l, 64+l, 96+l)
constexpr int ALN = 16;            // task bases are rounded down to 16 entries (16-byte flag copies)
constexpr int NG = CH / GE + 1;    // groups per task (+1: the task base is rounded down)
constexpr int MW = 4 * NG;         // mask words per task per mask (word j, bit l <-> entry 32j + l)
constexpr int SMALL = 32;  // segments of <= SMALL entries: one warp, one entry per lane (k_small)
constexpr int WARPS = 8;   // k2/k3 CTA size
constexpr int K1W = 4;     // k1 CTA size (warps); 4 CTAs/SM -> 16 warps, 128 registers
constexpr int SCAN_ITEMS = 8;  // plan_small (one launch) covers S < 8192
constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_TILE = SCAN_ITEMS * SCAN_THREADS;

struct StepP {
  Model md;
  int64_t ntask_max, max_mt;  // workspace capacities (guards against an inconsistent Q)
  const int64_t* pf_tab;
  const int32_t* pf_tab32;  // int32 copy when every entry fits (else nullptr)
  const int32_t* pf_fast;   // [PFT_N]: prefill_us(q + 1) for q < 2^17, values >= 2^30 stored as 2^30
  int32_t pt, bs, drop, offl, kdl, kpf;
  int64_t W, margin, Q;
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
  int32_t* task_seg;   // [#tasks]
  int64_t* scan_tmp;   // tile totals
  KI* cand;
  uint32_t *moff, *mdrop;
  int32_t *coff, *cdrop;
  int32_t* redo;       // [S]: short segments k_lane hands to k_small (outside its fast window)
  uint64_t bs_m, ab_m; // ceil(2^38 / block_tokens), ceil(2^38 / attention block b) (div_m)
  int32_t lane_ok;     // both divisors exact by div_m for every k_lane argument (< 2^17 + divisor)
  int32_t* redo_cnt;
  int* err;
};

__device__ __forceinline__ int64_t pf_of(const StepP& P, int32_t p) {
  if (p < P.pt) return P.pf_tab32 ? (int64_t)__ldg(P.pf_tab32 + p) : __ldg(P.pf_tab + p);
  const int64_t v = prefill_lat(P.md, (uint64_t)p);
  if (v < 0) { atomicOr(P.err, ERR_RANGE); return INT32_MAX; }
  return v;
}

// ---------------------------------------------------------------- planning (two scans) ------
__global__ void plan_counts(StepP P) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s > P.S) return;
  if (s == P.S) {
    if (P.seg_off[P.S] != P.Q) atomicOr(P.err, ERR_INVAL);
    *P.redo_cnt = 0;
    P.task_off[s] = 0;
    P.mtask_off[s] = 0;
    return;
  }
  const int64_t len = P.seg_off[s + 1] - P.seg_off[s];
  if (len < 0) atomicOr(P.err, ERR_INVAL);
  const int64_t nt = len <= SMALL ? 0 : len <= CH ? 1 : (len + CH - 1) / CH;  // small: k_small
  P.task_off[s] = nt;
  P.mtask_off[s] = nt > 1 ? nt : 0;
}

// block-local exclusive scan of (a, b) over tiles of SCAN_TILE; tile totals to tmp
__global__ void __launch_bounds__(SCAN_THREADS) scan_tiles(int64_t* a, int64_t* b, int64_t n, int64_t* tmp) {
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

__global__ void scan_add(StepP P, int64_t n, const int64_t* tmp) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t t = i / SCAN_TILE;
  P.task_off[i] += tmp[2 * t];
  P.mtask_off[i] += tmp[2 * t + 1];
}

__global__ void fill_task_seg(StepP P) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < P.S;
       s += (int64_t)gridDim.x * blockDim.x) {
    for (int64_t t = P.task_off[s]; t < P.task_off[s + 1] && t < P.ntask_max; t++)
      P.task_seg[t] = (int32_t)s;
  }
}

// two-launch planner for S >= SCAN_TILE: plan_tiles counts every segment's tasks from seg_off and
// scans them tile-locally (tile totals to scan_tmp); plan_fix adds the sum of the preceding tile
// totals (read directly: at most PLAN_FIX_TILES tiles) and writes the task -> segment map
constexpr int64_t PLAN_FIX_TILES = 4096;
// tasks of segment s from its length (segments of <= SMALL entries have none: k_lane / k_small)
__device__ __forceinline__ int32_t tasks_of(int64_t len) {
  return len <= SMALL ? 0 : len <= CH ? 1 : (int32_t)((len + CH - 1) / CH);
}
// One tile of SCAN_TILE = 8192 segments per CTA, warp w owning segments [w*256, w*256 + 256) of the
// tile with lane l at positions 32 i + l (coalesced loads and stores); tile-local sums fit int32
// (<= 8192 x 2^17 tasks).  SINGLE (S < SCAN_TILE): the final offsets and the task -> segment map in
// this one launch.  Otherwise tile-local exclusive offsets and tile totals (scan_tmp) for plan_fix.
template <bool SINGLE>
__global__ void __launch_bounds__(SCAN_THREADS) plan_tile(StepP P) {
  __shared__ int32_t sa[SCAN_THREADS / 32], sb[SCAN_THREADS / 32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int64_t tb = blockIdx.x * (int64_t)SCAN_TILE + w * 256 + l;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *P.redo_cnt = 0;
    if (P.seg_off[P.S] != P.Q) atomicOr(P.err, ERR_INVAL);
  }
  int64_t lo[SCAN_ITEMS + 1];
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) lo[i] = P.seg_off[min(tb + 32 * i, (int64_t)P.S)];
  int32_t na[SCAN_ITEMS], nb[SCAN_ITEMS];
  bool bad = false;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    const int64_t s = tb + 32 * i;
    const int64_t hi = P.seg_off[min(s + 1, (int64_t)P.S)];  // (the next lane's lo: an L1 hit)
    const int64_t len = hi - lo[i];
    bad |= s < P.S && len < 0;
    na[i] = s < P.S ? tasks_of(len) : 0;
    nb[i] = na[i] > 1 ? na[i] : 0;
  }
  if (bad) atomicOr(P.err, ERR_INVAL);
  int32_t ea[SCAN_ITEMS], eb[SCAN_ITEMS], ca = 0, cb = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    const int32_t ia = warp_incl_scan(na[i]), ib = warp_incl_scan(nb[i]);
    ea[i] = ca + ia - na[i];
    eb[i] = cb + ib - nb[i];
    ca += __shfl_sync(FULL, ia, 31);
    cb += __shfl_sync(FULL, ib, 31);
  }
  if (l == 0) { sa[w] = ca; sb[w] = cb; }
  __syncthreads();
  if (w == 0) {
    const int32_t x = sa[l], y = sb[l];
    const int32_t xi = warp_incl_scan(x), yi = warp_incl_scan(y);
    sa[l] = xi - x;
    sb[l] = yi - y;
    if (!SINGLE && l == 31) { P.scan_tmp[2 * blockIdx.x] = xi; P.scan_tmp[2 * blockIdx.x + 1] = yi; }
  }
  __syncthreads();
  const int64_t wa = sa[w], wb = sb[w];
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    const int64_t s = tb + 32 * i;
    if (s <= P.S) {
      const int64_t t0 = wa + ea[i];
      P.task_off[s] = t0;
      P.mtask_off[s] = wb + eb[i];
      if (SINGLE)
        for (int64_t t = t0; t < t0 + na[i] && t < P.ntask_max; t++) P.task_seg[t] = (int32_t)s;
    }
  }
}
__global__ void __launch_bounds__(SCAN_THREADS) plan_fix(StepP P) {
  __shared__ int64_t ra[SCAN_THREADS / 32], rb[SCAN_THREADS / 32];
  int64_t pa = 0, pb = 0;  // totals of the tiles before this one
  for (int64_t t = threadIdx.x; t < blockIdx.x; t += SCAN_THREADS) {
    pa += P.scan_tmp[2 * t];
    pb += P.scan_tmp[2 * t + 1];
  }
  pa = warp_sum(pa);
  pb = warp_sum(pb);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { ra[w] = pa; rb[w] = pb; }
  __syncthreads();
  pa = 0;
  pb = 0;
  for (int i = 0; i < SCAN_THREADS / 32; i++) { pa += ra[i]; pb += rb[i]; }
  // nothing before this tile and no task in it (every segment short: the usual LP queue): its
  // tile-local offsets are already the global ones and there is no task to map
  if (pa == 0 && pb == 0 && P.scan_tmp[2 * blockIdx.x] == 0) return;
  const int64_t tb = blockIdx.x * (int64_t)SCAN_TILE + w * 256 + l;
  // all loads first (clamped indices, no control flow between them), then the stores
  int64_t ta[SCAN_ITEMS], tm[SCAN_ITEMS], lo[SCAN_ITEMS], hi[SCAN_ITEMS];
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    const int64_t s = min(tb + 32 * i, (int64_t)P.S);
    ta[i] = P.task_off[s];
    tm[i] = P.mtask_off[s];
    lo[i] = P.seg_off[s];
    hi[i] = P.seg_off[min(s + 1, (int64_t)P.S)];
  }
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    const int64_t s = tb + 32 * i;
    if (s <= P.S) {
      const int64_t t0 = ta[i] + pa;
      P.task_off[s] = t0;
      P.mtask_off[s] = tm[i] + pb;
      const int32_t nt = s < P.S ? tasks_of(hi[i] - lo[i]) : 0;
      for (int64_t t = t0; t < t0 + nt && t < P.ntask_max; t++) P.task_seg[t] = (int32_t)s;
    }
  }
}

// ----------------------------------------------------------- Algorithm 1 over a sorted list --
// a[] holds the smallest live entries in (key, pos) order.  Writes admitted positions and the
// batch latency, returns k; `adm[r]` tells each lane which of its elements were admitted.
// TBT residual C of segment s (G22): tbt_slo - decode-only latency, or +inf without decodes
__device__ __forceinline__ int64_t seg_tbt_budget(const StepP& P, int64_t s) {
  const int64_t Bd = P.dcnt[s];
  if (Bd <= 0) return INF64;
  if (P.dctx[s] < Bd) atomicOr(P.err, ERR_INVAL);  // every context lhat >= 1 (oracle: same error)
  const int64_t d = lat_decode(P.md, (uint64_t)Bd, (uint64_t)P.dctx[s]);
  if (d < 0) { atomicOr(P.err, ERR_RANGE); return INF64; }
  return P.tbt[s] - d;
}

__device__ __forceinline__ int finalize_segment(const StepP& P, int64_t s, const KI (&a)[KPL],
                                                 bool (&adm)[KPL]) {
  const int lane = lane_id();
  const int64_t lo = P.seg_off[s];
  const int64_t N = P.bN[s], M = P.bM[s];
  int64_t R = P.bR[s];
  if (R > ASC_MAX_BATCH) { atomicOr(P.err, ERR_RANGE); R = ASC_MAX_BATCH; }
  const int64_t Bd = P.dcnt[s], sl = Bd > 0 ? P.dctx[s] : 0;  // no decodes: no context (oracle)
  const int64_t C = seg_tbt_budget(P, s);
  int32_t p[KPL];
  int64_t ct = 0, cb = 0, cc = 0;
  int k = 0;
  bool go = true;
#pragma unroll
  for (int r = 0; r < KPL; r++) {
    adm[r] = false;
    p[r] = 0;
  }
#pragma unroll
  for (int r = 0; r < KPL; r++) {
    if (!go) break;
    const bool valid = a[r].i != INF32;
    p[r] = valid ? __ldg(P.eff + a[r].i) : 0;
    const int64_t pf = valid ? pf_of(P, p[r]) : 0;
    const int64_t bl = valid ? (int64_t)((p[r] + P.bs) / P.bs) : 0;
    const int64_t St = ct + warp_incl_scan((int64_t)p[r]);
    const int64_t Sb = cb + warp_incl_scan(bl);
    const int64_t Sc = cc + warp_incl_scan(pf);
    const int pos = r * 32 + lane;
    const bool ok = valid && St < N && Sb < M && Sc < C && pos < R;
    const uint32_t m = __ballot_sync(FULL, ok);
    const int cnt = (m == FULL) ? 32 : (__ffs(~m) - 1);
    adm[r] = lane < cnt;
    k += cnt;
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
  if (k > 0) {
    sp = warp_sum(sp);
    sp2 = warp_sum(sp2);
    spc = warp_sum(spc);
  }
  if (lane == 0) {
    P.admit_cnt[s] = k;
    int64_t l = 0;
    if (k > 0 || Bd > 0) {
      l = k ? lat_us(P.md, (uint64_t)k, sp, sp2, spc, (uint64_t)Bd, (uint64_t)sl)
            : lat_decode(P.md, (uint64_t)Bd, (uint64_t)sl);
      if (l < 0) atomicOr(P.err, ERR_RANGE);
    }
    P.blat[s] = l;
  }
  return k;
}

// expand linear-layout mask words (word j, bit l <-> entry b4 + 32j + l) into id-ascending output
// indices starting at out[base]; returns the new base.  Each word's set lanes store their entries
// at consecutive ranks (one coalesced store per word, no staging ring).
__device__ __forceinline__ int64_t expand_groups(const uint32_t* words, int ng, int64_t b4,
                                                 int32_t* out, int64_t base) {
  const int lane = lane_id();
  const uint32_t lt = lanemask_lt(), bit = 1u << lane;
  int32_t* op = out + base;
  const int32_t e00 = (int32_t)b4 + lane;
  for (int g = 0; g < ng; g++) {
    const uint4 wv = *reinterpret_cast<const uint4*>(words + 4 * g);  // words 4g..4g+3
    if ((wv.x | wv.y | wv.z | wv.w) == 0) continue;
    const int32_t e0 = e00 + g * GE;
    if (wv.x & bit) op[__popc(wv.x & lt)] = e0;
    op += __popc(wv.x);
    if (wv.y & bit) op[__popc(wv.y & lt)] = e0 + 32;
    op += __popc(wv.y);
    if (wv.z & bit) op[__popc(wv.z & lt)] = e0 + 64;
    op += __popc(wv.z);
    if (wv.w & bit) op[__popc(wv.w & lt)] = e0 + 96;
    op += __popc(wv.w);
  }
  return base + (int64_t)(op - (out + base));
}

__device__ __forceinline__ void clear_admitted(uint32_t* words, int64_t loc) {
  atomicAnd(&words[loc >> 5], ~(1u << (loc & 31)));
}

struct Grp {  // one lane's 4 entries of a group: l, 32 + l, 64 + l, 96 + l
  int64_t dl[4];
  int32_t p[4];
  uint32_t f[4];
};

// one lane's entries gb + 32u + lane of the group starting at gb, bounds-checked (tails, generic path)
__device__ __forceinline__ void load_grp_s(const StepP& P, int64_t gb, Grp& g) {
  const int lane = lane_id();
#pragma unroll
  for (int u = 0; u < 4; u++) {
    const int64_t e = gb + 32 * u + lane;
    const bool in = e >= 0 && e < P.Q;
    g.dl[u] = in ? P.dl[e] : 0;
    g.p[u] = in ? P.eff[e] : 1;
    g.f[u] = in ? (uint32_t)P.fl[e] : 0u;
  }
}

// ---- cp.async staging: each lane copies its own 4 entries of a 128-entry group into a per-warp
// shared-memory ring (deadline 32 B, eff 16 B, flags 4 B per lane); no registers are held for
// data in flight and no cross-lane synchronisation is needed (a lane reads only what it copied).
#ifndef ASC_K1_NST
#define ASC_K1_NST 2
#endif
#ifndef ASC_K1_MINB
#define ASC_K1_MINB 4
#endif
constexpr int NST = ASC_K1_NST;  // pipeline stages per warp
struct Stage {
  longlong2 dl[2 * 32];  // lane l: dl[2l], dl[2l+1]
  int4 eff[32];
  uint32_t fl[32];
};

__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __noinline__ int64_t pf_slow(const StepP& P, int32_t p) {
  const int64_t v = prefill_lat(P.md, (uint64_t)p);
  if (v < 0) { atomicOr(P.err, ERR_RANGE); return INT32_MAX; }
  return v;
}

// k1 shared memory: per-warp staging rings (which also hold task_generic's candidate buffer), per-warp
// packed candidate buffers, and the per-warp masks of the enabled lists only
static_assert(sizeof(Stage) * NST >= sizeof(KI) * 160, "task_generic's buffer reuses the staging ring");
template <bool DROP, bool OFFL>
struct K1L {
  static constexpr size_t OFF_BUF = sizeof(Stage) * K1W * NST;
  static constexpr size_t OFF_OFF = OFF_BUF + sizeof(uint64_t) * K1W * 160;
  static constexpr size_t OFF_DROP = OFF_OFF + (OFFL ? 4 * K1W * MW : 0);
  static constexpr size_t SMEM = OFF_DROP + (DROP ? 4 * K1W * MW : 0);
};

// ---- budget-aware streaming selection (fast path).  A candidate packs into one uint64 whose
// unsigned order is the (key, index) order: ((key32 + 2^31) << 32) | (task-local index << 17) | (p - 1),
// p = the entry's effective prompt (<= 2^17).  The list is the warp's sorted 128 smallest
// candidates (position r*32 + lane in a[r]); the low field holds p - 1.  Algorithm 1 admits the longest prefix
// whose running sums of tokens, blocks and prefill µs stay strictly below N, M, C (and at most R
// entries), so after every merge the threshold moves to the first list position j whose running
// sums already reach a budget: the true prefix sum at any later key is at least the list's at j,
// so no entry above that element can be admitted, while the element itself (the first entry
// Algorithm 1 rejects) stays in the list.  Every entry of rank <= the first rejected one survives,
// which is all finalize_segment / k2 read.
constexpr int PK_LOC = 17;                          // bits of p below the local index
constexpr uint64_t PK_PMASK = (1ull << PK_LOC) - 1;
constexpr int32_t PFT_N = 1 << PK_LOC;              // fast table entries (p = 1 .. 2^17)
static_assert(PFT_N == ASC_PF_FAST_N, "fast table size");

struct TopKBud {
  uint64_t a[KPL];
  uint64_t thr;
  int cnt, kpos;
  bool any;
  uint64_t* buf;  // 320 slots in shared memory (per warp); at most 159 are used
  int32_t N, M, bs;
  int64_t C;
  const int32_t* tab;

  __device__ __forceinline__ void init(uint64_t* sbuf, int kpos_, int32_t N_, int32_t M_, int64_t C_,
                                       int32_t bs_, const int32_t* tab_) {
#pragma unroll
    for (int r = 0; r < KPL; r++) a[r] = PK_INF;
    thr = PK_INF;
    cnt = 0;
    kpos = kpos_;
    any = false;
    buf = sbuf;
    N = N_; M = M_; C = C_; bs = bs_; tab = tab_;
  }
  __device__ __forceinline__ void bitonic_merge() {
    const int l = lane_id();
#pragma unroll
    for (int j = KPL / 2; j > 0; j >>= 1) {
#pragma unroll
      for (int r = 0; r < KPL; r++) {
        if ((r & j) == 0) {
          const uint64_t x = a[r], y = a[r | j];
          a[r] = x < y ? x : y;
          a[r | j] = x < y ? y : x;
        }
      }
    }
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
      const bool lower = (l & j) == 0;
#pragma unroll
      for (int r = 0; r < KPL; r++) a[r] = pk_keep(a[r], __shfl_xor_sync(FULL, a[r], j), lower);
    }
  }
  __device__ __forceinline__ uint64_t at(int pos) const {
    const int r = pos >> 5;
    uint64_t x = a[0];
#pragma unroll
    for (int q = 1; q < KPL; q++) if (q == r) x = a[q];
    return __shfl_sync(FULL, x, pos & 31);
  }
  // first list position whose running (tokens, blocks, µs) reach (N, M, C), capped at kpos
  __device__ __forceinline__ int budget_pos() const {
    int pos = kpos;
    int32_t ct = 0, cb = 0;
    int64_t cc = 0;
    for (int r = 0; r < KPL && r * 32 <= pos; r++) {
      uint64_t x = a[0];
#pragma unroll
      for (int q = 1; q < KPL; q++) if (q == r) x = a[q];
      const bool valid = x != PK_INF;
      const int32_t q = (int32_t)(x & PK_PMASK);  // effective prompt - 1
      const int32_t p = valid ? q + 1 : 0;
      const int32_t bl = valid ? (p + bs) / bs : 0;
      const int64_t pf = valid ? (int64_t)__ldg(tab + q) : 0;
      const int32_t St = ct + warp_incl_scan(p);
      const int32_t Sb = cb + warp_incl_scan(bl);
      const int64_t Sc = cc + warp_incl_scan(pf);
      const uint32_t m = __ballot_sync(FULL, valid && (St >= N || Sb >= M || Sc >= C));
      if (m) return min(pos, r * 32 + __ffs(m) - 1);
      ct = __shfl_sync(FULL, St, 31);
      cb = __shfl_sync(FULL, Sb, 31);
      cc = __shfl_sync(FULL, Sc, 31);
    }
    return pos;
  }
  __device__ __forceinline__ void merge_sorted32(uint64_t y) {
    if (any) {
      const uint64_t br = __shfl_sync(FULL, y, 31 - lane_id());
      a[KPL - 1] = a[KPL - 1] < br ? a[KPL - 1] : br;
      bitonic_merge();
    } else {
      a[0] = y;
      any = true;
    }
    thr = at(budget_pos());
  }
  // merge the first 32 buffered candidates, then keep only the rest still below the new threshold
  __device__ __forceinline__ void flush32() {
    __syncwarp();
    const uint64_t y = buf[lane_id()];
    __syncwarp();
    merge_sorted32(sort32_pk(y));
    int nc = 0;
    for (int c0 = 32; c0 < cnt; c0 += 32) {
      const int j = c0 + lane_id();
      const uint64_t x = j < cnt ? buf[j] : PK_INF;
      const bool keep = x < thr;
      const uint32_t m = __ballot_sync(FULL, keep);  // also orders the read before the writes
      if (keep) buf[nc + __popc(m & lanemask_lt())] = x;
      nc += __popc(m);
    }
    cnt = nc;
    __syncwarp();
  }
  __device__ __forceinline__ void append(uint64_t x, bool c) {
    const uint32_t m = __ballot_sync(FULL, c);
    if (c) buf[cnt + __popc(m & lanemask_lt())] = x;
    cnt += __popc(m);
  }
  __device__ __forceinline__ void drain() {
    while (cnt >= 32) flush32();
  }
  __device__ __forceinline__ void finish() {
    drain();
    if (cnt > 0) {
      __syncwarp();
      const uint64_t y = lane_id() < cnt ? buf[lane_id()] : PK_INF;
      __syncwarp();
      cnt = 0;
      merge_sorted32(sort32_pk(y));
    }
  }
};

struct TaskCtx {  // per-task constants (uniform across the warp)
  int64_t s, lo, b, e_end, b4, now, othr;
  int32_t ng, vlo, vhi, kpos;
};

// Generic exact path: 64-bit keys and deadlines.  Used for a task whose deadlines or prefill
// latencies fall outside the 32-bit window of the fast path (or with an int64 latency table).
template <bool DROP, bool OFFL>
__device__ __noinline__ void task_generic(const StepP& P, const TaskCtx& t, KI* sbuf, uint32_t* m_off,
                                          uint32_t* m_drop, KI* out_a) {
  const int lane = lane_id();
  TopKStream<KPL> st;
  st.init(sbuf, t.kpos);
  const bool select = t.kpos >= 0;
  bool bad = false, rng = false;
  for (int g = 0; g < t.ng; g++) {
    const int64_t gb = t.b4 + (int64_t)g * GE;
    Grp cur;
    load_grp_s(P, gb, cur);
    const int32_t r0 = g * GE + lane;  // entry u of this lane: r0 + 32u (task-local), gb + lane + 32u
    KI x[4];
    bool cnd[4];
    uint32_t mo_w = 0, md_w = 0;
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const bool v = r0 + 32 * u >= t.vlo && r0 + 32 * u < t.vhi;
      const uint32_t f = cur.f[u];
      const int32_t pu = cur.p[u];
      bad |= v && pu < 1;
      rng |= v && pu >= (1 << 24);  // eff_prompt bound (keeps Σp² of a batch far from 2^64)
      int64_t pf = 0;
      if (v) {
        if (pu >= 1 && pu < P.pt) pf = P.pf_tab32 ? (int64_t)__ldg(P.pf_tab32 + pu) : __ldg(P.pf_tab + pu);
        else pf = pf_slow(P, pu < 1 ? 1 : pu);
      }
      if (P.pfout && v) {
        bad |= pf > INT32_MAX;
        __stcs(P.pfout + gb + lane + 32 * u, (int32_t)pf);
      }
      const bool dropped = DROP && v && !(f & 1u) && t.now > cur.dl[u];
      const bool off = OFFL && v && !dropped && !(f & 3u) && cur.dl[u] - pf <= t.othr;
      const uint32_t md = __ballot_sync(FULL, dropped), mo = __ballot_sync(FULL, off);
      md_w = lane == u ? md : md_w;
      mo_w = lane == u ? mo : mo_w;
      const int64_t spf = P.kpf > 0 ? pf : (P.kpf < 0 ? -pf : 0);
      x[u] = KI{(P.kdl ? cur.dl[u] : 0) + spf, (int32_t)(gb + lane + 32 * u)};
      cnd[u] = select && v && !dropped && ki_less(x[u], st.thr);
    }
    if (lane < 4) {
      if (DROP) m_drop[4 * g + lane] = md_w;
      if (OFFL) m_off[4 * g + lane] = mo_w;
    }
    if (__any_sync(FULL, cnd[0] | cnd[1] | cnd[2] | cnd[3])) {
#pragma unroll
      for (int u = 0; u < 4; u++) st.append(x[u], cnd[u]);
      st.drain();
    }
  }
  if (__any_sync(FULL, bad) && lane == 0) atomicOr(P.err, ERR_INVAL);
  if (__any_sync(FULL, rng) && lane == 0) atomicOr(P.err, ERR_RANGE);
  if (select) st.finish();
#pragma unroll
  for (int r = 0; r < KPL; r++) out_a[r] = st.top.a[r];
  __syncwarp();
}

constexpr int64_t WIN = int64_t(1) << 30;  // fast-path window: |deadline - now| < 2^30 us, pf < 2^30

// Fast path of one task: 32-bit arithmetic relative to `now`.  With d = deadline - now, each
// entry computes d' = d + 2^30 as the low word of one 64-bit add; the task is exact in 32 bits when
// every d' lies in [0, 2^31) (|d| <= 2^30 µs), every p in [1, 2^17] and every prefill below 2^30 µs.
// Those conditions are OR-accumulated (4 words per lane) and tested once at the end; a task that
// fails them is redone by task_generic.  Returns false in that case.
template <bool VEC, bool DROP, bool OFFL>
__device__ __forceinline__ bool task_fast(const StepP& P, const TaskCtx& t, Stage (&stg)[NST], uint64_t* sbuf,
                                          uint32_t* m_off, uint32_t* m_drop, int64_t Cb, KI (&top)[KPL]) {
  const int lane = lane_id();
  const int ng = t.ng;
  const int64_t b4 = t.b4;
  const bool select = t.kpos >= 0;
  const int64_t nowc = WIN - t.now;  // d' = deadline + nowc
  // offload iff deadline - prefill_us <= now + W_hp + margin  <=>  d' - pf <= othr1
  const int32_t othr1 = (int32_t)min(P.W + P.margin + WIN, (int64_t)INT32_MAX);
  const int32_t dmask = P.kdl ? -1 : 0;
  const int32_t kpf = P.kpf;
  const int32_t* __restrict__ tab = P.pf_fast;
  const bool has_pfout = P.pfout != nullptr;
  TopKBud st;
  st.init(sbuf, t.kpos, P.bN[t.s], P.bM[t.s], Cb, P.bs, tab);
  uint32_t accH = 0, accL = 0, accQ = 0, accF = 0;
  const uint32_t vspan = (uint32_t)(t.vhi - t.vlo);
  // groups [0, nfull) lie entirely below Q: staged through shared memory without bounds tests
  int nfull = 0;
  if (VEC) {
    const int64_t nf = (P.Q - b4) / GE;
    nfull = (int)(nf < ng ? nf : ng);
  }
  const int64_t* gdl = P.dl + b4 + 4 * lane;
  const int32_t* gef = P.eff + b4 + 4 * lane;
  const uint8_t* gfl = P.fl + b4 + 16 * (lane & 7);  // lanes 0-7 copy the group's 128 flag bytes
  const int l = lane;
#pragma unroll
  for (int q = 0; q < NST - 1; q++) {
    if (q < nfull) {
      cp_async16(&stg[q].dl[2 * l], gdl + q * GE);
      cp_async16(&stg[q].dl[2 * l + 1], gdl + q * GE + 2);
      cp_async16(&stg[q].eff[l], gef + q * GE);
      if (l < 8) cp_async16(&stg[q].fl[4 * l], gfl + q * GE);
    }
    cp_commit();
  }
  for (int g = 0; g < ng; g++) {
    const int gi = g + NST - 1;
    __syncwarp();  // every lane is done reading the slot lanes 0-7 refill next
    if (gi < nfull) {
      Stage& sg = stg[gi % NST];
      cp_async16(&sg.dl[2 * l], gdl + gi * GE);
      cp_async16(&sg.dl[2 * l + 1], gdl + gi * GE + 2);
      cp_async16(&sg.eff[l], gef + gi * GE);
      if (l < 8) cp_async16(&sg.fl[4 * l], gfl + gi * GE);
    }
    cp_commit();
    const int64_t gb = b4 + (int64_t)g * GE;  // this lane's entries: gb + lane + 32u
    Grp cur;
    if (g < nfull) {
      cp_wait<NST - 1>();
      __syncwarp();  // every lane reads entries other lanes copied
      const Stage& sg = stg[g % NST];
      const int64_t* sd = reinterpret_cast<const int64_t*>(sg.dl);
      const int32_t* se = reinterpret_cast<const int32_t*>(sg.eff);
      const uint8_t* sf = reinterpret_cast<const uint8_t*>(sg.fl);
#pragma unroll
      for (int u = 0; u < 4; u++) {  // consecutive lanes, consecutive entries: conflict-free
        cur.dl[u] = sd[32 * u + l];
        cur.p[u] = se[32 * u + l];
        cur.f[u] = sf[32 * u + l];
      }
    } else {
      load_grp_s(P, gb, cur);
    }
    const int32_t r0 = g * GE + lane;            // task-local index of this lane's entry u: r0 + 32u
    const uint32_t l0 = (uint32_t)r0 << PK_LOC;
    // candidates are filtered on the packed word's high half (the key) only: key <= the
    // threshold's key keeps every entry below the threshold (plus, rarely, ties above it, which the
    // merge sorts past it); the full word is packed only for the candidates, in the append below
    const uint32_t thr_hi = (uint32_t)(st.thr >> 32);
    uint32_t kw[4];
    bool cnd[4];
    int32_t pfv[4];
    uint32_t mo[4], md[4];
    auto body = [&](auto interior) {
      constexpr bool IN = decltype(interior)::value;
#pragma unroll
      for (int u = 0; u < 4; u++) {  // branch-free: every lane runs the same instructions
        const bool v = IN || (uint32_t)(r0 + 32 * u - t.vlo) < vspan;
        const int64_t dd = cur.dl[u] + nowc;
        const uint32_t lo1 = (uint32_t)dd, hi1 = (uint32_t)((uint64_t)dd >> 32);
        const int32_t q = cur.p[u] - 1;
        const int32_t pf = __ldg(tab + ((uint32_t)q & (uint32_t)PK_PMASK));  // unsigned: one IMAD.WIDE
        accH |= v ? hi1 : 0u;
        accL |= v ? lo1 : 0u;
        accQ |= v ? (uint32_t)q : 0u;
        accF |= v ? (uint32_t)pf : 0u;
        pfv[u] = pf;
        if (!IN && has_pfout && v) __stcs(P.pfout + gb + l + 32 * u, pf);
        const int32_t d1 = (int32_t)lo1;  // deadline - now + 2^30
        const uint32_t f = cur.f[u];
        const bool dropped = DROP && v && !(f & 1u) && d1 < (int32_t)WIN;
        const bool off = OFFL && v && !dropped && !(f & 3u) && d1 - pf <= othr1;
        if (DROP) md[u] = __ballot_sync(FULL, dropped);
        if (OFFL) mo[u] = __ballot_sync(FULL, off);
        const int32_t key1 = (d1 & dmask) + kpf * pf;  // kdl * d' + kpf * pf, branch-free
        kw[u] = (uint32_t)key1 ^ 0x80000000u;
        cnd[u] = select && v && !dropped && kw[u] <= thr_hi;
      }
    };
    if (r0 - lane >= t.vlo && r0 - lane + GE <= t.vhi) {
      body(std::true_type{});
      if (has_pfout)
#pragma unroll
        for (int u = 0; u < 4; u++) __stcs(P.pfout + gb + l + 32 * u, pfv[u]);  // coalesced per u
    } else {
      body(std::false_type{});
    }
    if (lane == 0) {  // the group's 4 ballot words
      if (DROP) *reinterpret_cast<uint4*>(m_drop + 4 * g) = make_uint4(md[0], md[1], md[2], md[3]);
      if (OFFL) *reinterpret_cast<uint4*>(m_off + 4 * g) = make_uint4(mo[0], mo[1], mo[2], mo[3]);
    }
    if (__any_sync(FULL, cnd[0] | cnd[1] | cnd[2] | cnd[3])) {
#pragma unroll
      for (int u = 0; u < 4; u++)
        st.append(((uint64_t)kw[u] << 32) |
                      (uint64_t)(l0 + ((uint32_t)(32 * u) << PK_LOC) + ((uint32_t)(cur.p[u] - 1) & (uint32_t)PK_PMASK)),
                  cnd[u]);
      st.drain();
    }
  }
  cp_wait<0>();
  __syncwarp();
  const bool ok = accH == 0 && !(accL & 0x80000000u) && !(accQ & ~(uint32_t)PK_PMASK) && !(accF & 0xC0000000u);
  if (!__all_sync(FULL, ok)) return false;
  if (select) st.finish();
  const int64_t kbase = P.kdl ? t.now - WIN : 0;  // key = kbase + key1
#pragma unroll
  for (int r = 0; r < KPL; r++) {
    const uint64_t x = st.a[r];
    top[r] = x == PK_INF ? ki_inf()
                         : KI{kbase + (int64_t)(int32_t)((uint32_t)(x >> 32) ^ 0x80000000u),
                              (int32_t)(b4 + (int64_t)((uint32_t)x >> PK_LOC))};
  }
  return true;
}

// TAB: 0 = int64 latency table (generic path only), 1 = int32 table (fast path)
template <bool VEC, int TAB, bool DROP, bool OFFL>
__global__ void __launch_bounds__(K1W * 32, ASC_K1_MINB) k1_tasks(const __grid_constant__ StepP P) {
  using L = K1L<DROP, OFFL>;
  extern __shared__ __align__(16) unsigned char k1_smem[];  // L::SMEM bytes (dynamic)
  auto& s_stage = *reinterpret_cast<Stage(*)[K1W][NST]>(k1_smem);
  auto& sbuf = *reinterpret_cast<uint64_t(*)[K1W][160]>(k1_smem + L::OFF_BUF);
  auto& s_off = *reinterpret_cast<uint32_t(*)[K1W][MW]>(k1_smem + L::OFF_OFF);
  auto& s_drop = *reinterpret_cast<uint32_t(*)[K1W][MW]>(k1_smem + L::OFF_DROP);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntasks = min(P.task_off[P.S], P.ntask_max);
  for (int64_t task = blockIdx.x * (int64_t)K1W + w; task < ntasks;
       task += (int64_t)gridDim.x * K1W) {
    TaskCtx t;
    t.s = P.task_seg[task];
    const int64_t s = t.s;
    const int64_t c = task - P.task_off[s];
    const int64_t nt = P.task_off[s + 1] - P.task_off[s];
    t.lo = P.seg_off[s];
    const int64_t hi = P.seg_off[s + 1];
    t.b = t.lo + c * CH;
    t.e_end = min(hi, t.b + CH);
    t.b4 = t.b & ~int64_t(ALN - 1);
    t.ng = (int)((t.e_end - t.b4 + GE - 1) / GE);
    t.vlo = (int32_t)(t.b - t.b4);
    t.vhi = (int32_t)(t.e_end - t.b4);
    t.now = P.now[s];
    t.othr = t.now + P.W + P.margin;  // offload iff deadline - prefill_us <= othr
    // Algorithm 1 can admit at most min(R, N-1, M-1) entries (strict budgets, costs >= 1): only
    // that many smallest keys are needed, so the running threshold sits at that position
    int64_t kneed = P.bR[s];
    kneed = kneed < 32 * KPL ? kneed : 32 * KPL;
    kneed = kneed < (int64_t)P.bN[s] - 1 ? kneed : (int64_t)P.bN[s] - 1;
    kneed = kneed < (int64_t)P.bM[s] - 1 ? kneed : (int64_t)P.bM[s] - 1;
    const int64_t Cb = seg_tbt_budget(P, s);  // every prefill costs >= 1 µs
    kneed = kneed < Cb - 1 ? kneed : Cb - 1;
    t.kpos = kneed > 0 ? (int)kneed - 1 : -1;
    const int64_t b4 = t.b4, lo = t.lo;
    const int ng = t.ng;
    KI top[KPL];
    bool fast_ok = (TAB == 1);
    if (TAB == 1)
      fast_ok = task_fast<VEC, DROP, OFFL>(P, t, s_stage[w], sbuf[w], s_off[w], s_drop[w], Cb, top);
    if (!fast_ok) {
      KI tmp[KPL];
      task_generic<DROP, OFFL>(P, t, reinterpret_cast<KI*>(&s_stage[w][0]), s_off[w], s_drop[w], tmp);
#pragma unroll
      for (int r = 0; r < KPL; r++) top[r] = tmp[r];
    }
    __syncwarp();
    if (nt == 1) {
      bool adm[KPL];
      finalize_segment(P, s, top, adm);
      // an admitted request is not offloaded (only unscheduled requests)
#pragma unroll
      for (int r = 0; r < KPL; r++)
        if (OFFL && adm[r]) clear_admitted(s_off[w], top[r].i - b4);
      __syncwarp();
      const int64_t no = OFFL ? expand_groups(s_off[w], ng, b4, P.off_idx, lo) : lo;
      const int64_t nd = DROP ? expand_groups(s_drop[w], ng, b4, P.drop_idx, lo) : lo;
      if (lane == 0) { P.off_cnt[s] = (int32_t)(no - lo); P.drop_cnt[s] = (int32_t)(nd - lo); }
    } else {
      const int64_t mt = P.mtask_off[s] + c;
      if (mt >= P.max_mt) continue;
      KI* cd = P.cand + mt * (32 * KPL);
#pragma unroll
      for (int r = 0; r < KPL; r++) cd[r * 32 + lane] = top[r];
      int32_t co = 0, cdp = 0;
      for (int j = lane; j < MW; j += 32) {
        const uint32_t mo = (OFFL && j < 4 * ng) ? s_off[w][j] : 0u;
        const uint32_t mdp = (DROP && j < 4 * ng) ? s_drop[w][j] : 0u;
        P.moff[mt * MW + j] = mo;
        P.mdrop[mt * MW + j] = mdp;
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

// Segments of at most SMALL entries (short queues: the common case of a real LP instance): one
// warp per segment, one entry per lane — a1 (table), a2 key, a3 as one 32-wide bitonic sort of
// (key, position), a4 as a strict prefix-sum scan in sorted order, a5 ballots in position order,
// a6 from the admitted moments.  Same outputs as k1 (SURVEY row S, 10^6 x 32).
#ifndef ASC_KS_MINB
#define ASC_KS_MINB 3
#endif
// Inputs of one short segment, loaded one segment ahead (the loop below is a chain of dependent
// loads per segment: seg_off -> entries -> latency table; prefetching overlaps it with the work)
struct SmallIn {
  int64_t lo, n, dl, now, sl, tbt;
  int32_t p, R, Bd, N, M;
  uint32_t f;
};
__device__ __forceinline__ void small_load(const StepP& P, int64_t s, SmallIn& x) {
  const int lane = lane_id();
  x.lo = 0; x.n = -1;
  if (s >= P.S) return;
  x.lo = P.seg_off[s];
  x.n = P.seg_off[s + 1] - x.lo;
  x.dl = 0; x.p = 1; x.f = 0;
  if (x.n > SMALL || x.n < 0) return;
  if (lane < x.n) {
    const int64_t e = x.lo + lane;
    x.dl = __ldcs(P.dl + e);
    x.p = __ldcs(P.eff + e);
    x.f = __ldcs(P.fl + e);
  }
  x.now = P.now[s];
  x.R = P.bR[s];
  x.Bd = P.dcnt[s];
  x.sl = x.Bd > 0 ? P.dctx[s] : 0;  // dec_ctx_sum is ignored without decodes
  x.tbt = P.tbt[s];
  x.N = P.bN[s];
  x.M = P.bM[s];
}

// LIST: the segments k_lane handed back (P.redo[0 .. *P.redo_cnt)); otherwise every segment
template <bool LIST>
__global__ void __launch_bounds__(256, ASC_KS_MINB) k_small(const __grid_constant__ StepP P) {
  const int lane = lane_id();
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nseg = LIST ? (int64_t)*P.redo_cnt : (int64_t)P.S;
  auto seg_at = [&](int64_t i) -> int64_t { return LIST ? (i < nseg ? (int64_t)P.redo[i] : (int64_t)P.S) : i; };
  int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  SmallIn nx;
  small_load(P, seg_at(i), nx);
  for (; i < nseg; i += nw) {
    const int64_t s = seg_at(i);
    const SmallIn cu = nx;
    small_load(P, seg_at(i + nw), nx);  // next segment's inputs in flight during this one
    const int64_t lo = cu.lo, n = cu.n;
    if (n > SMALL || n < 0) continue;  // k1's, or invalid (the planner flags it)
    const bool v = lane < n;
    const int64_t e = lo + lane;
    const int64_t dl = cu.dl;
    const int32_t p = cu.p;
    const uint32_t f = cu.f;
    bool bad = v && p < 1;
    if (__any_sync(FULL, v && p >= (1 << 24)) && lane == 0) atomicOr(P.err, ERR_RANGE);
    const int64_t pf = v ? pf_of(P, p < 1 ? 1 : p) : 0;
    if (P.pfout && v) {
      bad |= pf > INT32_MAX;
      __stcs(P.pfout + e, (int32_t)pf);
    }
    if (__any_sync(FULL, bad) && lane == 0) atomicOr(P.err, ERR_INVAL);
    const int64_t now = cu.now;
    const bool dropped = P.drop && v && !(f & 1u) && now > dl;
    // value function (FCFS: 0, ties by position); dropped and empty lanes sort last
    const int64_t key = (P.kdl ? dl : 0) + (P.kpf > 0 ? pf : (P.kpf < 0 ? -pf : 0));
    // a3: one 32-wide bitonic sort of (key, position).  Keys within 2^31 µs of the base (now for
    // the deadline-based policies) pack with the position into one uint64 (two shuffles per step);
    // otherwise the (int64 key, position) pairs are sorted directly.
    const bool lv = v && !dropped;
    const int64_t rel = key - (P.kdl ? now : 0);
    KI x;
    if (__all_sync(FULL, !lv || (rel >= -(int64_t(1) << 26) && rel < (int64_t(1) << 26) - 1))) {
      // keys within 2^26 µs of the base: (key, position) in one uint32 (one shuffle per step)
      const uint32_t pk = lv ? ((uint32_t)(rel + (int64_t(1) << 26)) << 5) | (uint32_t)lane : 0xffffffffu;
      const uint32_t y = sort32_u32(pk);
      x.i = y == 0xffffffffu ? INF32 : (int32_t)(y & 31u);
      x.k = 0;  // unused below
    } else if (__all_sync(FULL, !lv || (rel >= INT32_MIN && rel <= INT32_MAX))) {
      const uint64_t pk = lv ? ((uint64_t)((uint32_t)(int32_t)rel ^ 0x80000000u) << 32) | (uint32_t)lane : PK_INF;
      const uint64_t y = sort32_pk(pk);
      x.i = y == PK_INF ? INF32 : (int32_t)(uint32_t)y;
      x.k = 0;  // unused below
    } else {
      x = sort32(lv ? KI{key, lane} : ki_inf());
    }
    const bool live = x.i != INF32;
    const int src = live ? x.i : 0;
    const int32_t ps = __shfl_sync(FULL, p, src);
    const int64_t pfs = __shfl_sync(FULL, pf, src);
    const int64_t bls = live ? (int64_t)(((uint32_t)ps + (uint32_t)P.bs) / (uint32_t)P.bs) : 0;  // ps < 2^31
    // Algorithm 1 lines 5-13: strict budgets N (tokens), M (blocks), C (TBT residual), R (requests)
    int64_t R = cu.R;
    if (R > ASC_MAX_BATCH) { if (lane == 0) atomicOr(P.err, ERR_RANGE); R = ASC_MAX_BATCH; }
    const int64_t Bd = cu.Bd, sl = cu.sl;
    if (lane == 0 && Bd > 0 && sl < Bd) atomicOr(P.err, ERR_INVAL);  // every lhat >= 1
    // a6 for every prefix at once: lane j evaluates the batch {first j sorted entries} ∪ D
    // (Eq. 3-5 from the exclusive prefix moments).  Lane 0 is the decode-only batch, whose
    // latency also gives the TBT residual C (G22); the admitted batch is lane k's — one fused
    // evaluation instead of two sequential ones.  Only the lanes used may raise ERR_RANGE.
    const uint64_t qv = live ? (uint64_t)ps : 0ull;
    const uint64_t q2 = qv * qv;
    const uint64_t qc = live ? qv * (uint64_t)(((uint32_t)ps + (uint32_t)P.md.b - 1u) / (uint32_t)P.md.b) : 0ull;  // ps < 2^31
    const uint64_t isp = (uint64_t)warp_incl_scan((int64_t)qv);
    const uint64_t isp2 = (uint64_t)warp_incl_scan((int64_t)q2);
    const uint64_t ispc = (uint64_t)warp_incl_scan((int64_t)qc);
    const int64_t lj = (lane > 0 || Bd > 0)
                           ? lat_us(P.md, (uint64_t)lane, isp - qv, isp2 - q2, ispc - qc, (uint64_t)Bd, (uint64_t)sl)
                           : 0;
    int64_t C = INF64;
    const int64_t d = __shfl_sync(FULL, lj, 0);
    if (Bd > 0) {
      if (d < 0 && lane == 0) atomicOr(P.err, ERR_RANGE);
      C = cu.tbt - d;
    }
    const int64_t St = warp_incl_scan(live ? (int64_t)ps : (int64_t)0);
    const int64_t Sb = warp_incl_scan(bls);
    const int64_t Sc = warp_incl_scan(live ? pfs : (int64_t)0);
    const bool ok = live && St < (int64_t)cu.N && Sb < (int64_t)cu.M && Sc < C && lane < R;
    const uint32_t m = __ballot_sync(FULL, ok);
    const int k = (m == FULL) ? 32 : (__ffs(~m) - 1);
    const bool adm = lane < k;
    if (adm) P.admit_idx[lo + lane] = (int32_t)(lo + x.i);
    const uint32_t amask = __reduce_or_sync(FULL, adm ? (1u << x.i) : 0u);
    int64_t lk = __shfl_sync(FULL, lj, k & 31);  // k < 32: lane k's prefix
    if (k == 32)                                  // every lane admitted: the full sums (lane 31's inclusive)
      lk = lat_us(P.md, 32, __shfl_sync(FULL, isp, 31), __shfl_sync(FULL, isp2, 31), __shfl_sync(FULL, ispc, 31),
                  (uint64_t)Bd, (uint64_t)sl);
    // a5: offload (non-admitted, never prefilled, not on an HP) and drop lists in position order
    const bool off = P.offl && v && !dropped && !((amask >> lane) & 1u) && !(f & 3u) &&
                     dl - now <= pf + P.W + P.margin;
    const uint32_t mo = __ballot_sync(FULL, off), md = __ballot_sync(FULL, dropped);
    if (off) P.off_idx[lo + __popc(mo & lanemask_lt())] = (int32_t)e;
    if (dropped) P.drop_idx[lo + __popc(md & lanemask_lt())] = (int32_t)e;
    if (lane == 0) {
      P.admit_cnt[s] = k;
      P.off_cnt[s] = __popc(mo);
      P.drop_cnt[s] = __popc(md);
      int64_t l = 0;
      if (k > 0 || Bd > 0) {
        l = lk;
        if (l < 0) atomicOr(P.err, ERR_RANGE);
      }
      P.blat[s] = l;
    }
  }
}

// ------------------------------------------------------------- k_lane: one THREAD per segment --
// Short segments (<= SMALL entries: SURVEY row S's 10^6 x 32 shape, the queue of a real LP
// instance).  A warp takes 32 consecutive segments, stages their contiguous entry range into shared
// memory with coalesced 16-byte cp.async copies, and then every lane decides its own segment
// serially (§5): a1 (prefill table), the key (a2), the drop / offload predicates as
// 32-bit position masks (a5), a3 as a 32-input bitonic network over packed (key, position) words
// held in registers, a4 as a strict prefix scan in key order with early exit, and a6 twice
// (decode-only batch for the TBT residual C, then the admitted batch).  No shuffles and one fp64
// evaluation per batch instead of one per prefix: about a tenth of k_small's instructions.
// A lane reads its entries rotated by (lane mod n) so that equal-length neighbours hit distinct
// shared-memory banks.  Segments outside the fast window (p outside [1, 2^17], a prefill >= 2^30 µs,
// a live key more than 2^26 µs from now, R > ASC_MAX_BATCH, an invalid decode count / context) or
// in a group whose entry range exceeds the staging buffer go to P.redo; k_small<true> decides them
// (and raises their errors) afterwards.
constexpr int LW = 4;             // k_lane CTA size (warps); 4 CTAs/SM
constexpr int LCAP = 32 * SMALL;  // staged entries per warp (32 segments of <= SMALL)
struct __align__(16) LaneStage {
  int64_t dl[LCAP + 2];    // chunk-aligned copies (first chunk aligned down to 16 bytes); after
  int32_t eff[LCAP + 4];   // pass 1 the low word of dl[e] holds prefill_us of entry e
  uint8_t fl[LCAP + 16];
  uint64_t bar;            // mbarrier: completion of the group's bulk copies
};
static_assert(sizeof(int64_t) * (LCAP + 2) % 16 == 0 && sizeof(int32_t) * (LCAP + 4) % 16 == 0, "16-byte aligned rows");

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "LAB_WAIT%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// one TMA bulk copy (1-D, 16-byte aligned, size a multiple of 16) completing on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// Stage g[lo0, hi) into dst as 16-byte chunks from the aligned-down start a0 (returns a0): the chunks
// inside [0, Q) as ONE bulk copy issued by lane 0 (bytes added to *tx), the at most two chunks that
// cross the array ends element by element by the other lanes.
template <typename T>
__device__ __forceinline__ int64_t lane_stage(T* dst, const T* g, int64_t lo0, int64_t hi, int64_t Q,
                                              uint64_t* bar, unsigned* tx) {
  constexpr int K = 16 / sizeof(T);
  const int64_t a0 = lo0 - (int64_t)(((uintptr_t)(g + lo0) & 15) / sizeof(T));
  const int64_t nch = (hi - a0 + K - 1) / K;
  const int64_t c0 = a0 < 0 ? (-a0 + K - 1) / K : 0;           // first chunk with e >= 0
  int64_t c1 = (Q - a0) / K;                                     // chunks [c0, c1) end <= Q
  c1 = c1 < nch ? c1 : nch;
  const int lane = lane_id();
  if (c1 > c0) {
    if (lane == 0) bulk_g2s(dst + c0 * K, g + a0 + c0 * K, (unsigned)((c1 - c0) * 16), bar);
    *tx += (unsigned)((c1 - c0) * 16);
  }
  // boundary chunks [0, c0) and [t0, nch): element by element
  const int64_t t0 = c1 > c0 ? c1 : c0;
  const int hb = (int)(c0 < nch ? c0 : nch) * K, nb = hb + (int)(nch > t0 ? nch - t0 : 0) * K;
  for (int i = lane; i < nb; i += 32) {
    const int64_t x = i < hb ? (int64_t)i : t0 * K + (i - hb);  // element offset from a0
    const int64_t e = a0 + x;
    if (e >= 0 && e < Q) dst[x] = g[e];
  }
  return a0;
}

// per-segment inputs of k_lane, loaded (coalesced across the warp's 32 segments) while the entry
// range is still being staged
struct LaneSeg {
  int64_t now, sl, tbt;
  int32_t R, Bd, N, M;
};
__device__ __forceinline__ void lane_seg_load(const StepP& P, int64_t s, LaneSeg& x) {
  x.now = P.now[s];
  x.R = P.bR[s];
  x.Bd = P.dcnt[s];
  x.sl = P.dctx[s];
  x.tbt = P.tbt[s];
  x.N = P.bN[s];
  x.M = P.bM[s];
}
// x / d for 0 <= x < 2^38 / d by one multiply: m = ceil(2^38 / d) = (2^38 + e) / d with e < d, so
// x * m / 2^38 = x / d + x * e / (d * 2^38) and the error term stays below 1 / d (StepP::lane_div)
__device__ __forceinline__ uint32_t div_m(uint32_t x, uint64_t m) { return (uint32_t)(((uint64_t)x * m) >> 38); }

// decide segment s (entries [lo, lo + n), staged at st with chunk bases a0d / a0e / a0f); false if
// the segment is outside the fast window (nothing written yet).  F32: n == 32 (the row-S shape;
// warp-uniform), so the rotation is (j + lane) & 31 and no entry test is needed.  Every deadline is
// taken relative to now in 32 bits: d = deadline - now must lie in (-2^30, 2^30) (else: hand back),
// so d - pf, the key d*kdl + pf*kpf and the offload test are exact int32 arithmetic.
template <bool F32>
__device__ __forceinline__ bool lane_segment(const StepP& P, LaneStage& st, int64_t s, int64_t lo, int n,
                                             const LaneSeg& g, int64_t a0d, int64_t a0e, int64_t a0f) {
  const int32_t R = g.R, Bd = g.Bd;
  const int64_t sl = Bd > 0 ? g.sl : 0;  // dec_ctx_sum is ignored without decodes
  if (R > ASC_MAX_BATCH || Bd < 0 || (Bd > 0 && sl < Bd)) return false;
  const int64_t now = g.now;
  const int od = (int)(lo - a0d), oe = (int)(lo - a0e), of = (int)(lo - a0f);
  int32_t* pfs = reinterpret_cast<int32_t*>(st.dl);  // pf of entry j at pfs[2 * (od + j)]
  const int lane = lane_id();
  const int rot = F32 ? lane : (n > 0 ? lane % n : 0);
  auto slot = [&](int j) {  // rotated position of the j-th visit; 0 past the end (never used)
    if (F32) return (j + lane) & (SMALL - 1);
    int jj = j + rot;
    jj -= jj >= n ? n : 0;
    return j < n ? jj : 0;
  };
  // two halves of 16 entries: all 16 a1 table gathers of a half in flight at once (branch-free, no
  // dependence between entries), then the key, drop and offload candidates of that half (position
  // order is kept in the masks)
  constexpr int H = SMALL / 2;
  uint32_t a[SMALL];
  uint32_t dm = 0, om = 0, bad = 0, mxw = 0;
  const int32_t othr = (int32_t)max((int64_t)INT32_MIN, min((int64_t)INT32_MAX, P.W + P.margin));
  const bool kdl = P.kdl != 0, drop = P.drop != 0, offl = P.offl != 0;
  const int32_t kpf = P.kpf;
  int32_t pfv[H];
  if (F32 || n > 0) {  // (an empty segment reads nothing: its slot 0 is the next lane's entry)
#pragma unroll
  for (int h = 0; h < SMALL; h += H) {
#pragma unroll
    for (int j = h; j < h + H; j++) {
      const int32_t p = st.eff[oe + slot(j)];
      pfv[j - h] = __ldg(P.pf_fast + ((p - 1) & (PFT_N - 1)));
      if (F32 || j < n) bad |= (uint32_t)(p - 1) & ~(uint32_t)(PFT_N - 1);  // p outside [1, 2^17]
    }
#pragma unroll
    for (int j = h; j < h + H; j++) {
      const int jj = slot(j);
      const bool v = F32 || j < n;
      const int64_t d64 = st.dl[od + jj] - now;
      const int32_t d = (int32_t)d64, pf = pfv[j - h];
      const uint32_t f = st.fl[of + jj];
      // window (else hand back): d = deadline - now in [-2^30, 2^30) (d64 is d sign-extended, and
      // d + 2^30 < 2^31), pf < 2^26, the packed key field rel + 2^26 < 2^27 - 1; so d - pf and the
      // key are exact int32, 32 prefill times sum below 2^31, and the packed word of a live entry
      // is never the all-ones sentinel
      const uint32_t u = (uint32_t)((kdl ? d : 0) + kpf * pf + (1 << 26));
      if (v) {
        bad |= (uint32_t)(d64 >> 32) ^ (uint32_t)(d >> 31);
        mxw = max(mxw, max((uint32_t)(d + (1 << 30)) >> 4, (uint32_t)pf << 1));  // < 2^27 iff both in range
        mxw = max(mxw, u);
      }
      const bool dropped = v && drop && !(f & 1u) && d < 0;
      const bool offc = v && offl && !dropped && !(f & 3u) && d - pf <= othr;
      a[j] = (!v || dropped) ? 0xffffffffu : (u << 5) | (uint32_t)jj;
      if (F32) {  // bits in visit order; rotated to positions once below
        dm |= dropped ? (1u << j) : 0u;
        om |= offc ? (1u << j) : 0u;
      } else {
        dm |= (uint32_t)dropped << jj;
        om |= (uint32_t)offc << jj;
      }
      if (v)  // this entry's deadline is not read again: keep (pf, p) in its place (v: an empty
              // segment's slot 0 is the next lane's entry)
        reinterpret_cast<int2*>(st.dl)[od + jj] = make_int2(pf, st.eff[oe + jj]);
    }
  }
  }
  if (F32) {  // visit j is position (j + lane) & 31: rotate left by lane
    dm = __funnelshift_l(dm, dm, lane);
    om = __funnelshift_l(om, om, lane);
  }
  bad |= mxw >= (1u << 27) - 1 ? 1u : 0u;
  const bool ok = bad == 0;
  if (!ok) return false;
  // a3: ascending (key, position); dropped entries (all ones) sort last
#pragma unroll
  for (int k = 2; k <= SMALL; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
      for (int i = 0; i < SMALL; i++) {
        const int l = i ^ j;
        if (l > i) {
          const uint32_t x = a[i], y = a[l];
          const bool up = (i & k) == 0;
          a[i] = up ? min(x, y) : max(x, y);
          a[l] = up ? max(x, y) : min(x, y);
        }
      }
  // C: TBT residual after the decode-only batch (G22)
  int64_t C = INF64, d = 0;
  if (Bd > 0) {
    d = lat_us(P.md, 0, 0, 0, 0, (uint64_t)Bd, (uint64_t)sl);
    if (d < 0) atomicOr(P.err, ERR_RANGE);
    C = g.tbt - d;
  }
  // the sorted keys go to this lane's own eff slots (its p values now sit beside pf), so that
  // Algorithm 1's loop below can index them without unrolling
  uint32_t* ks = reinterpret_cast<uint32_t*>(st.eff) + oe;
#pragma unroll
  for (int j = 0; j < SMALL; j++)
    if (F32 || j < n) ks[slot(j)] = a[j];
  // a4: Algorithm 1 lines 5-13, strict budgets in key order (prefix sums of tokens, blocks and
  // prefill µs strictly below N, M, C; at most R).  Σpf < 2^31, so the µs budget compares in 32
  // bits against C clamped to [0, 2^32 - 1].  The next entry is fetched before the current one is
  // tested.
  const int32_t N = g.N, M = g.M;
  const uint32_t bs = (uint32_t)P.bs, ab1 = (uint32_t)P.md.b - 1u;
  const uint32_t Cc = C <= 0 ? 0u : (C >= (int64_t)0xffffffff ? 0xffffffffu : (uint32_t)C);
  const int2* ent = reinterpret_cast<const int2*>(st.dl) + od;  // (pf, p) by position
  const int jmax = min(F32 ? SMALL : n, (int)max(R, 0));
  int32_t St = 0, Sb = 0;
  uint32_t Sc = 0, sp = 0;
  int k = 0;
  uint32_t am = 0;
  uint64_t sp2 = 0, spc = 0;
  // (a sentinel's position field is read as entry 0: never outside this lane's segment)
  // two entries in flight ahead of the one being tested (the key -> entry loads are dependent)
  uint32_t xn = jmax > 0 ? ks[slot(0)] : 0xffffffffu, xn2 = jmax > 1 ? ks[slot(1)] : 0xffffffffu;
  int2 en = ent[xn == 0xffffffffu ? 0u : (xn & 31u)], en2 = ent[xn2 == 0xffffffffu ? 0u : (xn2 & 31u)];
  int32_t* adm = P.admit_idx + lo;
#pragma unroll 2
  for (int j = 0; j < jmax; j++) {
    const uint32_t x = xn;
    const int2 e = en;
    xn = xn2;
    en = en2;
    if (j + 2 < jmax) {
      xn2 = ks[slot(j + 2)];
      en2 = ent[xn2 == 0xffffffffu ? 0u : (xn2 & 31u)];
    }
    if (x == 0xffffffffu) break;
    const uint32_t p = (uint32_t)e.y;
    St += (int32_t)p;
    Sb += (int32_t)div_m(p + bs, P.bs_m);
    Sc += (uint32_t)e.x;
    if (!(St < N && Sb < M && Sc < Cc)) break;
    const uint32_t pos = x & 31u;
    adm[j] = (int32_t)(lo + pos);
    am |= 1u << pos;
    k = j + 1;
    sp += p;
    sp2 += (uint64_t)p * p;
    spc += (uint64_t)p * div_m(p + ab1, P.ab_m);
  }
  // a6: the hybrid batch {admitted} + {decodes}
  int64_t l = 0;
  if (k > 0 || Bd > 0) {
    l = k ? lat_us(P.md, (uint64_t)k, (uint64_t)sp, sp2, spc, (uint64_t)Bd, (uint64_t)sl) : d;
    if (l < 0) atomicOr(P.err, ERR_RANGE);
  }
  // a5: offload (not admitted) and drop lists in ascending position
  uint32_t mo = om & ~am;
  int co = 0, cd = 0;
  while (mo) {
    P.off_idx[lo + co++] = (int32_t)(lo + __ffs(mo) - 1);
    mo &= mo - 1;
  }
  while (dm) {
    P.drop_idx[lo + cd++] = (int32_t)(lo + __ffs(dm) - 1);
    dm &= dm - 1;
  }
  if (P.pfout)
    for (int j = 0; j < n; j++) P.pfout[lo + j] = pfs[2 * (od + j)];
  P.admit_cnt[s] = k;
  P.off_cnt[s] = co;
  P.drop_cnt[s] = cd;
  P.blat[s] = l;
  return true;
}

#ifndef ASC_KL_MINB
#define ASC_KL_MINB 4
#endif
// the general (n != 32) case out of line: its register pressure stays out of the F32 path's
__device__ __noinline__ bool lane_segment_any(const StepP& P, LaneStage& st, int64_t s, int64_t lo, int n,
                                              const LaneSeg& g, int64_t a0d, int64_t a0e, int64_t a0f) {
  return lane_segment<false>(P, st, s, lo, n, g, a0d, a0e, a0f);
}

__global__ void __launch_bounds__(LW * 32, ASC_KL_MINB) k_lane(const __grid_constant__ StepP P) {
  extern __shared__ __align__(16) unsigned char kl_smem[];
  LaneStage& st = reinterpret_cast<LaneStage*>(kl_smem)[threadIdx.x >> 5];
  const int lane = lane_id();
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t ng = ((int64_t)P.S + 31) >> 5;
  if (lane == 0) mbar_init(&st.bar);
  __syncwarp();
  unsigned phase = 0;
  for (int64_t gi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; gi < ng; gi += nw) {
    const int64_t s = gi * 32 + lane;
    const bool has = s < P.S;
    int64_t lo = 0, hi = 0;
    LaneSeg sg{};
    if (has) {
      lo = P.seg_off[s];
      hi = P.seg_off[s + 1];
      lane_seg_load(P, s, sg);  // in flight during the staging below
    }
    const int last = (int)min((int64_t)31, (int64_t)P.S - 1 - gi * 32);
    const int64_t lo0 = __shfl_sync(FULL, lo, 0), hiN = __shfl_sync(FULL, hi, last);
    const bool fits = P.lane_ok && hiN >= lo0 && hiN - lo0 <= LCAP && lo0 >= 0 && hiN <= P.Q;  // uniform
    // n > SMALL: k1's segment; a non-monotone seg_off is flagged by the planner
    const bool mine = has && hi - lo >= 0 && hi - lo <= SMALL;
    int64_t a0d = 0, a0e = 0, a0f = 0;
    if (fits) {
      // the previous group's generic-proxy accesses to the buffer come before the async writes
      if (lane == 0) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      unsigned tx = 0;
      a0d = lane_stage(st.dl, P.dl, lo0, hiN, P.Q, &st.bar, &tx);
      a0e = lane_stage(st.eff, P.eff, lo0, hiN, P.Q, &st.bar, &tx);
      a0f = lane_stage(st.fl, P.fl, lo0, hiN, P.Q, &st.bar, &tx);
      if (lane == 0) mbar_arrive_tx(&st.bar, tx);
      mbar_wait(&st.bar, phase);
      phase ^= 1u;
    }
    __syncwarp();
    bool redo = mine;
    const bool all32 = __all_sync(FULL, !has || hi - lo == SMALL);
    if (mine && fits && lo >= lo0 && hi <= hiN)
      redo = all32 ? !lane_segment<true>(P, st, s, lo, SMALL, sg, a0d, a0e, a0f)
                   : !lane_segment_any(P, st, s, lo, (int)(hi - lo), sg, a0d, a0e, a0f);
    const uint32_t m = __ballot_sync(FULL, redo);
    if (m) {
      int base = 0;
      if (lane == 0) base = atomicAdd(P.redo_cnt, __popc(m));
      base = __shfl_sync(FULL, base, 0);
      if (redo) P.redo[base + __popc(m & lanemask_lt())] = (int32_t)s;
    }
    __syncwarp();  // the staging buffer is refilled next
  }
}

__global__ void __launch_bounds__(WARPS * 32) k2_segments(const __grid_constant__ StepP P) {
  __shared__ KI lists[WARPS][32 * KPL];
  __shared__ int64_t segs[WARPS * 32];
  __shared__ int nseg;
  if (P.mtask_off[P.S] == 0) return;  // no segment has more than one task (the common case)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // find this CTA's multi-task segments up to 256 at a time (most segments have one task or
  // none); chunks shrink with S so that few large segments still spread over the CTAs
  int64_t chunk = P.S / gridDim.x;
  chunk = chunk < 1 ? 1 : (chunk > WARPS * 32 ? WARPS * 32 : chunk);
  for (int64_t base = (int64_t)blockIdx.x * chunk; base < P.S; base += (int64_t)gridDim.x * chunk) {
    if (threadIdx.x == 0) nseg = 0;
    __syncthreads();
    const int64_t s0 = base + threadIdx.x;
    if (threadIdx.x < chunk && s0 < P.S && P.task_off[s0 + 1] - P.task_off[s0] > 1)
      segs[atomicAdd(&nseg, 1)] = s0;
    __syncthreads();
    const int cnt = nseg;
  for (int q = 0; q < cnt; q++) {
    const int64_t s = segs[q];
    const int64_t nt = P.task_off[s + 1] - P.task_off[s];
    const int64_t m0 = P.mtask_off[s];
    if (m0 + nt > P.max_mt) continue;
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
          const int64_t e = A.a[r].i;
          const int64_t t = (e - lo) / CH;
          const int64_t b4 = (lo + t * CH) & ~int64_t(ALN - 1);
          const int64_t loc = e - b4;
          const uint32_t bit = 1u << (loc & 31);
          const uint32_t old = atomicAnd(&P.moff[(m0 + t) * MW + (loc >> 5)], ~bit);
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
    __syncthreads();  // segs is rewritten by the next round
  }
}

// K3P warps per multi-task task, each expanding a contiguous quarter of its 128-entry groups (more
// independent warps in flight than one per task): a part's output offset is the task's (k2's scan)
// plus the set bits of the task's earlier mask words
constexpr int K3P = 4;
constexpr int K3W = (NG + K3P - 1) / K3P;  // groups per part
__global__ void __launch_bounds__(WARPS * 32) k3_expand(const __grid_constant__ StepP P) {
  __shared__ __align__(16) uint32_t s_words[WARPS][2][4 * K3W];
  if (P.mtask_off[P.S] == 0) return;  // no multi-task segment
  const int w = threadIdx.x >> 5, lane = lane_id();
  const int64_t ntasks = min(P.task_off[P.S], P.ntask_max);
  for (int64_t item = blockIdx.x * (int64_t)WARPS + w; item < ntasks * K3P;
       item += (int64_t)gridDim.x * WARPS) {
    const int64_t task = item / K3P;
    const int part = (int)(item % K3P);
    const int64_t s = P.task_seg[task];
    const int64_t nt = P.task_off[s + 1] - P.task_off[s];
    if (nt <= 1) continue;
    const int64_t c = task - P.task_off[s];
    const int64_t mt = P.mtask_off[s] + c;
    if (mt >= P.max_mt) continue;
    const int64_t lo = P.seg_off[s], hi = P.seg_off[s + 1];
    const int64_t b = lo + c * CH;
    const int64_t e_end = min(hi, b + CH);
    const int64_t b4 = b & ~int64_t(ALN - 1);
    const int ng = (int)((e_end - b4 + GE - 1) / GE);
    const int g0 = part * K3W, g1 = min(ng, g0 + K3W);
    if (g0 >= g1) continue;
    const uint32_t* wo = P.moff + mt * MW;
    const uint32_t* wd = P.mdrop + mt * MW;
    int32_t po = 0, pd = 0;  // set bits of the words before this part
    for (int j = lane; j < 4 * g0; j += 32) {
      po += __popc(wo[j]);
      pd += __popc(wd[j]);
    }
    po = warp_sum(po);
    pd = warp_sum(pd);
    // this part's mask words to shared memory in one coalesced pass: expand_groups reads one
    // 16-byte word group per iteration, a dependent global load each time otherwise
    const int nw4 = 4 * (g1 - g0);
    for (int j = lane; j < nw4; j += 32) {
      s_words[w][0][j] = wo[4 * g0 + j];
      s_words[w][1][j] = wd[4 * g0 + j];
    }
    __syncwarp();
    const int64_t bg = b4 + (int64_t)g0 * GE;
    expand_groups(s_words[w][0], g1 - g0, bg, P.off_idx, lo + P.coff[mt] + po);
    expand_groups(s_words[w][1], g1 - g0, bg, P.drop_idx, lo + P.cdrop[mt] + pd);
    __syncwarp();
  }
}

template <bool VEC, int TAB, bool DROP, bool OFFL>
void launch_k1_t(unsigned grid, size_t, cudaStream_t sm, const StepP& P) {
  constexpr size_t SMEM = K1L<DROP, OFFL>::SMEM;
  auto* k = k1_tasks<VEC, TAB, DROP, OFFL>;
  // attributes and the resident-CTA cap once per device (host work between launches is GPU idle
  // time of every call)
  static std::mutex mu;
  static unsigned caps[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  unsigned cap = 0;
  {
    std::lock_guard<std::mutex> g(mu);
    cap = dev < 64 ? caps[dev] : 0;
    if (!cap) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
      // shared memory for ASC_K1_MINB resident CTAs and no more: the rest of the unified L1 caches
      // the prefill table the per-entry a1 lookups gather from
      const int carve = (int)((ASC_K1_MINB * (SMEM + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024));
      cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve < 100 ? carve : 100);
      int sms = 148, nb = ASC_K1_MINB;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, K1W * 32, SMEM);
      cap = (unsigned)(sms * (nb > 0 ? nb : 1));
      if (dev < 64) caps[dev] = cap;
    }
  }
  k<<<grid < cap ? grid : cap, K1W * 32, SMEM, sm>>>(P);
}

template <int TAB, bool DROP, bool OFFL>
void launch_k1_v(bool vec, unsigned grid, size_t dsm, cudaStream_t sm, const StepP& P) {
  if (vec) launch_k1_t<true, TAB, DROP, OFFL>(grid, dsm, sm, P);
  else launch_k1_t<false, TAB, DROP, OFFL>(grid, dsm, sm, P);
}

template <int TAB>
void launch_k1_d(int variant, unsigned grid, size_t dsm, cudaStream_t sm, const StepP& P) {
  const bool vec = variant & 1, drop = variant & 8, offl = variant & 16;
  if (drop && offl) launch_k1_v<TAB, true, true>(vec, grid, dsm, sm, P);
  else if (drop) launch_k1_v<TAB, true, false>(vec, grid, dsm, sm, P);
  else if (offl) launch_k1_v<TAB, false, true>(vec, grid, dsm, sm, P);
  else launch_k1_v<TAB, false, false>(vec, grid, dsm, sm, P);
}

void launch_k1(int variant, unsigned grid, size_t dsm, cudaStream_t sm, const StepP& P) {
  launch_k1_d<1>(variant, grid, dsm, sm, P);  // the fast table always exists; task_generic covers the rest
}

}  // namespace

namespace asc {

asc_status launch_schedule_step(asc_ctx* c, const asc_step_in* in, asc_step_out* out, int64_t Q) {
  const int32_t S = in->S;
  const int64_t max_mt = 2 * (Q / CH) + 2;
  const int64_t ntask_max = (int64_t)S + Q / CH + 1;
  const int64_t ntile = (S + 1 + SCAN_TILE - 1) / SCAN_TILE;
  size_t need = 0;
  need += 2 * (size_t)(S + 1) * 8 + 2 * (size_t)ntile * 8 + (size_t)ntask_max * 4 + 8192;
  need += (size_t)max_mt * (32 * KPL) * sizeof(KI) + (size_t)max_mt * MW * 8 + (size_t)max_mt * 8 + 8192;
  need += (size_t)(S + 1) * 4 + 1024;  // k_lane's hand-back list
  asc_status st = ensure_ws(c, need);
  if (st) return st;
  Arena ar{c->ws, c->ws_cap};
  StepP P;
  P.md = c->md;
  P.ntask_max = ntask_max;
  P.max_mt = max_mt;
  P.pf_tab = c->d_pf_tab;
  P.pf_tab32 = c->d_pf_tab32;
  P.pf_fast = c->d_pf_fast;
  P.pt = c->pt_size;
  P.bs = c->cfg.topo.block_tokens;
  P.drop = c->cfg.flags.drop;
  P.offl = (c->cfg.flags.offload && c->cfg.topo.n_hp >= 1) ? 1 : 0;
  // value function as key = kdl*deadline + kpf*prefill_us (FCFS: 0 = position order)
  switch (c->cfg.flags.policy) {
    case ASC_POLICY_EDF_LAXITY: P.kdl = 1; P.kpf = -1; break;
    case ASC_POLICY_EDF_DEADLINE: P.kdl = 1; P.kpf = 0; break;
    case ASC_POLICY_SJF: P.kdl = 0; P.kpf = 1; break;
    case ASC_POLICY_LJF: P.kdl = 0; P.kpf = -1; break;
    default: P.kdl = 0; P.kpf = 0; break;
  }
  P.W = c->w_hp;
  P.margin = c->cfg.flags.offload_margin_us;
  P.Q = Q;
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
  P.task_seg = ar.take<int32_t>(ntask_max);
  P.cand = ar.take<KI>(max_mt * 32 * KPL);
  P.moff = ar.take<uint32_t>(max_mt * MW);
  P.mdrop = ar.take<uint32_t>(max_mt * MW);
  P.coff = ar.take<int32_t>(max_mt);
  P.cdrop = ar.take<int32_t>(max_mt);
  P.redo = ar.take<int32_t>(S > 0 ? S : 1);
  {  // div_m is exact for x < 2^38 / d; k_lane's arguments stay below 2^17 + d
    const uint64_t bsd = (uint64_t)P.bs, abd = (uint64_t)P.md.b;
    P.bs_m = ((uint64_t(1) << 38) + bsd - 1) / bsd;
    P.ab_m = ((uint64_t(1) << 38) + abd - 1) / abd;
    P.lane_ok = bsd <= (1u << 16) && abd <= (1u << 16);
  }
  P.redo_cnt = ar.take<int32_t>(1);
  P.err = c->d_err;
  cudaStream_t sm = c->stream;
  g_prof.mark(1);
  int64_t launches = 0;
  const int dev_sms = c->sms;
  if (S + 1 <= SCAN_TILE) {
    plan_tile<true><<<1, SCAN_THREADS, 0, sm>>>(P);
    launches += 1;
  } else if (ntile <= PLAN_FIX_TILES) {
    plan_tile<false><<<ntile, SCAN_THREADS, 0, sm>>>(P);
    plan_fix<<<ntile, SCAN_THREADS, 0, sm>>>(P);
    launches += 2;
  } else {
    plan_counts<<<(S + 1 + 255) / 256, 256, 0, sm>>>(P);
    scan_tiles<<<ntile, SCAN_THREADS, 0, sm>>>(P.task_off, P.mtask_off, S + 1, P.scan_tmp);
    scan_totals<<<1, 32, 0, sm>>>(P.scan_tmp, ntile);
    scan_add<<<(S + 1 + 255) / 256, 256, 0, sm>>>(P, S + 1, P.scan_tmp);
    const int64_t gf = (S + 255) / 256;
    fill_task_seg<<<(unsigned)(gf < 4 * dev_sms ? (gf > 0 ? gf : 1) : 4 * dev_sms), 256, 0, sm>>>(P);
    launches += 5;
  }
  g_prof.mark(2);
  {  // a planner that failed to launch must not leave k1 reading an unscanned task map
    const cudaError_t pe = cudaGetLastError();
    if (pe != cudaSuccess) return cuda_check(c, pe, "schedule_step planner launch");
  }
  int64_t g1 = (ntask_max + K1W - 1) / K1W;  // clamped to the resident CTAs by launch_k1_t
  g1 = g1 < (int64_t)dev_sms * 32 ? g1 : (int64_t)dev_sms * 32;
  const bool vec = ((uintptr_t)in->deadline_us % 16 == 0) && ((uintptr_t)in->eff_prompt % 16 == 0) &&
                   ((uintptr_t)in->flags % 16 == 0) && ((uintptr_t)P.pfout % 16 == 0);
  const unsigned gk = (unsigned)(g1 > 0 ? g1 : 1);
  const int tab = P.pf_tab32 ? 1 : 0;
  const size_t dsm = 0;
  const int variant = (vec ? 1 : 0) | (tab << 1) | (P.drop ? 8 : 0) | (P.offl ? 16 : 0);
  cudaEventRecord(c->ev0, sm);
  launch_k1(variant, gk, dsm, sm, P);
  {
    const cudaError_t ke = cudaGetLastError();  // checked here: later runtime calls may not keep it
    if (ke != cudaSuccess) return cuda_check(c, ke, "schedule_step k1 launch");
  }
  cudaEventRecord(c->ev1, sm);
  c->timed = true;
  launches += 1;
  g_prof.mark(3);
  {  // short segments (after k1's timed bracket: k1 is the roofline kernel of row S's big shape):
     // k_lane decides them one per thread, k_small the ones it hands back
    constexpr size_t LSMEM = LW * sizeof(LaneStage);
    {
      static std::mutex mu;
      static uint64_t set = 0;  // devices whose k_lane attribute is set
      std::lock_guard<std::mutex> g(mu);
      if (c->device >= 64 || !(set >> c->device & 1)) {
        cudaFuncSetAttribute(k_lane, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LSMEM);
        if (c->device < 64) set |= uint64_t(1) << c->device;
      }
    }
    int64_t gl = (((int64_t)S + 31) / 32 + LW - 1) / LW;
    gl = gl < (int64_t)dev_sms * 4 ? gl : (int64_t)dev_sms * 4;  // one resident wave
    cudaEventRecord(c->ev2, sm);
    k_lane<<<(unsigned)(gl > 0 ? gl : 1), LW * 32, LSMEM, sm>>>(P);
    cudaEventRecord(c->ev3, sm);
    c->timed2 = true;
    int64_t gs = ((int64_t)S * 32 + 255) / 256;
    gs = gs < (int64_t)dev_sms * ASC_KS_MINB ? gs : (int64_t)dev_sms * ASC_KS_MINB;
    k_small<true><<<(unsigned)(gs > 0 ? gs : 1), 256, 0, sm>>>(P);
    launches += 2;
  }
  g_prof.mark(4);
  if (Q > CH) {
    int64_t g2 = S < (int64_t)dev_sms * 4 ? S : (int64_t)dev_sms * 4;
    k2_segments<<<(unsigned)(g2 > 0 ? g2 : 1), WARPS * 32, 0, sm>>>(P);
    int64_t g3 = (ntask_max * K3P + WARPS - 1) / WARPS;
    g3 = g3 < (int64_t)dev_sms * 8 ? g3 : (int64_t)dev_sms * 8;
    k3_expand<<<(unsigned)(g3 > 0 ? g3 : 1), WARPS * 32, 0, sm>>>(P);
    launches += 2;
  }
  c->last_kernel_launches = launches;
  const asc_status lst = cuda_check(c, cudaGetLastError(), "schedule_step launch");
  g_prof.mark(5);
  return lst;
}

}  // namespace asc
