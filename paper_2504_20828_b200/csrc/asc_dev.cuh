// asc_dev.cuh — device building blocks of the sm_100a hot path (no oracle code is shared).
//
//  * Model / lat_us: the performance model of PAPER.md Eq. 1-5 with the App. A GEMM
//    terms (Tables 3-4, Eq. 6-7), evaluated from per-batch integer moments
//    (B_p, Σp, Σp², Σp·⌈p/b⌉, B_d, Σl̂) so a batch of any size costs O(1) after a warp reduction.
//    F and M are exact uint64 (< 2^53); the fp64 regression uses explicit round-to-nearest
//    intrinsics in a fixed order (no FMA contraction) so the result is bitwise reproducible.
//  * WarpTopK: per-warp streaming selection of the K = 32*KPL smallest (key, idx) pairs, held as a
//    sorted list in registers (element e at lane e%32, register e/32), merged with bitonic
//    networks over warp shuffles.  Algorithm 1 only ever admits a prefix of at most R <= K
//    entries of the key order, so the K smallest entries are all it needs.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace asc {

constexpr int64_t INF64 = INT64_MAX;
constexpr int32_t INF32 = INT32_MAX;
constexpr uint64_t TWO53 = 1ull << 53;
constexpr uint32_t FULL = 0xffffffffu;

// error bits raised by kernels (ctx->dev_err)
constexpr int ERR_RANGE = 1;
constexpr int ERR_INVARIANT = 2;
constexpr int ERR_INVAL = 4;

struct Model {
  uint64_t n, s, L, d, b;
  uint64_t W;    // weights per layer (elements): 4h^2 + 2hm (read once per non-empty batch, G8)
  uint64_t FT;   // GEMM flops per token per layer: 4h^2 + 2hm (Tables 3-4 row sums)
  uint64_t MT;   // GEMM activation elements per token per layer: 8h + 2m
  // decode-only batches in closed form (exact integer identities of the expression below):
  // F = dF_bd*B_d + dF_sl*Σl̂,  M = dM_0 + dM_bd*B_d + dM_sl*Σl̂
  uint64_t dF_bd, dF_sl, dM_0, dM_bd, dM_sl;
  double c0, c1, c2, c3, c4, FH, MH;
};

// Eq. 4-5 + G17/G18 from exact integer F, M (< 2^53): fixed fp64 RN order, ceil to microseconds.
// Out of line: the two correctly rounded divisions expand to a long sequence, and one copy keeps
// the event-loop kernel inside the instruction cache.
// Eq. 4-5 in seconds, clamped at 0: the value lat_from_FM rounds.
static __device__ __forceinline__ double t_from_FM(const Model& md, uint64_t F, uint64_t M) {
  const double tM = __ddiv_rn(__ull2double_rn(M), md.MH);
  const double tF = __ddiv_rn(__ull2double_rn(F), md.FH);
  const double mx = (tM > tF) ? tM : tF;
  double t = __dmul_rn(md.c0, __dadd_rn(tM, tF));
  t = __dadd_rn(t, __dmul_rn(md.c1, mx));
  t = __dadd_rn(t, __dmul_rn(md.c2, tM));
  t = __dadd_rn(t, __dmul_rn(md.c3, tF));
  t = __dadd_rn(t, md.c4);
  if (!(t > 0.0)) t = 0.0;
  return t;
}
__device__ __forceinline__ int64_t us_of_t(double t) {  // G18 + G17
  const int64_t v = (int64_t)ceil(__dmul_rn(t, 1e6));
  return v < 1 ? 1 : v;
}
static __device__ __noinline__ int64_t lat_from_FM(const Model& md, uint64_t F, uint64_t M) {
  return us_of_t(t_from_FM(md, F, M));
}

// Decode-only batch of B_d requests with context sum sl (a2's TBT term, a6 for decode steps).
// The fp64 shadow below guards the uint64 products against wrapping (as wraps() does).
// INL: the fp64 evaluation inlined (one hot call site) instead of the shared out-of-line copy
template <bool INL = false>
__device__ __forceinline__ int64_t lat_decode(const Model& md, uint64_t Bd, uint64_t sl) {
  const uint64_t F = md.dF_bd * Bd + md.dF_sl * sl;
  const uint64_t M = md.dM_0 + md.dM_bd * Bd + md.dM_sl * sl;
  if (F >= TWO53 || M >= TWO53) return -1;
  const double bd = (double)Bd, s = (double)sl;
  if ((double)md.dF_bd * bd + (double)md.dF_sl * s >= 0x1p62 ||
      (double)md.dM_0 + (double)md.dM_bd * bd + (double)md.dM_sl * s >= 0x1p62) return -1;
  return INL ? us_of_t(t_from_FM(md, F, M)) : lat_from_FM(md, F, M);
}

// uint64 wrap guard: F and M are sums of products of non-negative integers, so no
// intermediate exceeds the final value; if the same expression evaluated in fp64 (relative error
// < 2^-40 here) stays below 2^62, the true values are below 2^63 and the uint64 results are exact.
// Otherwise the true F or M is far above 2^53 and the batch is out of range.  The inputs' own sums
// (Σp, Σp², ...) are bounded by the callers' validation (eff_prompt < 2^24, <= 128 requests).
__host__ __device__ inline bool wraps(const Model& md, uint64_t sp, uint64_t sp2, uint64_t spm /* 3 Σp⌈p/b⌉ */,
                                      uint64_t Bd, uint64_t sl, uint64_t G) {
  const double n = (double)md.n, s = (double)md.s, tok = (double)sp + (double)Bd;
  const double F = (double)md.L * (tok * (double)md.FT + n * (2.0 * s * (double)sp2 + 2.0 * s * (double)sl));
  const double M = (double)md.L * (double)md.d *
                   ((double)G * (double)md.W + tok * (double)md.MT +
                    n * (2.0 * s * (double)sp + s * (double)spm + 2.0 * s * (double)sl + 2.0 * s * (double)Bd));
  return F >= 0x1p62 || M >= 0x1p62;
}
__host__ __device__ inline bool wraps_chunked(const Model& md, uint64_t sc, uint64_t aF, uint64_t aM,
                                              uint64_t Bd, uint64_t sl, uint64_t G) {
  const double n = (double)md.n, s = (double)md.s, tok = (double)sc + (double)Bd;
  const double F = (double)md.L * (tok * (double)md.FT + n * (2.0 * s * (double)aF + 2.0 * s * (double)sl));
  const double M = (double)md.L * (double)md.d *
                   ((double)G * (double)md.W + tok * (double)md.MT +
                    n * (s * (double)aM + 2.0 * s * (double)sl + 2.0 * s * (double)Bd));
  return F >= 0x1p62 || M >= 0x1p62;
}

// Latency in integer microseconds of a batch given its integer moments (G17, G18).
// Returns -1 (and the caller raises ERR_RANGE) when F or M reaches 2^53.
template <bool INL = false>  // INL: the fp64 evaluation inlined (device), as lat_decode<true>
__host__ __device__ inline int64_t lat_us(const Model& md, uint64_t Bp, uint64_t sp, uint64_t sp2,
                                          uint64_t spc, uint64_t Bd, uint64_t sl) {
  const uint64_t tok = sp + Bd;
  const uint64_t G = (Bp + Bd) ? 1 : 0;
  const uint64_t attnF = md.n * (2 * md.s * sp2 + 2 * md.s * sl);
  const uint64_t attnM = md.n * (2 * md.s * sp + 3 * md.s * spc + 2 * md.s * sl + 2 * md.s * Bd);
  const uint64_t F = md.L * (tok * md.FT + attnF);
  const uint64_t M = md.L * (G * md.W + tok * md.MT + attnM) * md.d;
  if (F >= TWO53 || M >= TWO53 || wraps(md, sp, sp2, 3 * spc, Bd, sl, G)) return -1;
#ifdef __CUDA_ARCH__
  return INL ? us_of_t(t_from_FM(md, F, M)) : lat_from_FM(md, F, M);
#else
  volatile double tM = (double)M / md.MH;
  volatile double tF = (double)F / md.FH;
  const double mx = (tM > tF) ? tM : tF;
  volatile double t = md.c0 * (tM + tF);
  t = t + md.c1 * mx;
  t = t + md.c2 * tM;
  t = t + md.c3 * tF;
  t = t + md.c4;
  if (!(t > 0.0)) t = 0.0;
  volatile double t6 = t * 1e6;
  const int64_t v = (int64_t)ceil(t6);
  return v < 1 ? 1 : v;
#endif
}

__host__ __device__ inline uint64_t ceil_div_u(uint64_t x, uint64_t y) { return (x + y - 1) / y; }

// App. A.4 hybrid batch with chunked prefill (readings G48) from per-batch sums over its nch
// chunks (chunk = l tokens already prefilled + c new): sc = Σc, aF = Σ(l·c + c²),
// aM = Σ(2l + 3c⌈l/b⌉ + 2c + 3c⌈c/b⌉); plus B_d decodes with context sum sl.  Whole prompts
// (l = 0) give exactly lat_us's F and M.
__device__ __forceinline__ int64_t lat_chunked(const Model& md, uint64_t nch, uint64_t sc,
                                               uint64_t aF, uint64_t aM, uint64_t Bd, uint64_t sl) {
  const uint64_t tok = sc + Bd;
  const uint64_t G = (nch + Bd) ? 1 : 0;
  const uint64_t attnF = md.n * (2 * md.s * aF + 2 * md.s * sl);
  const uint64_t attnM = md.n * (md.s * aM + 2 * md.s * sl + 2 * md.s * Bd);
  const uint64_t F = md.L * (tok * md.FT + attnF);
  const uint64_t M = md.L * (G * md.W + tok * md.MT + attnM) * md.d;
  if (F >= TWO53 || M >= TWO53 || wraps_chunked(md, sc, aF, aM, Bd, sl, G)) return -1;
  return lat_from_FM(md, F, M);
}

// Standalone prefill latency of one prompt of p tokens (a1).
__host__ __device__ inline int64_t prefill_lat(const Model& md, uint64_t p) {
  return lat_us(md, 1, p, p * p, p * ceil_div_u(p, md.b), 0, 0);
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  uint64_t z = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) { T w = __shfl_xor_sync(FULL, v, o); v = w < v ? w : v; }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) { T w = __shfl_xor_sync(FULL, v, o); v = w > v ? w : v; }
  return v;
}
// 32-bit integer reductions are one REDUX instruction each (sm_80+)
__device__ __forceinline__ int32_t warp_sum(int32_t v) { return __reduce_add_sync(FULL, v); }
__device__ __forceinline__ uint32_t warp_sum(uint32_t v) { return __reduce_add_sync(FULL, v); }
__device__ __forceinline__ int32_t warp_min(int32_t v) { return __reduce_min_sync(FULL, v); }
__device__ __forceinline__ uint32_t warp_min(uint32_t v) { return __reduce_min_sync(FULL, v); }
__device__ __forceinline__ int32_t warp_max(int32_t v) { return __reduce_max_sync(FULL, v); }
__device__ __forceinline__ uint32_t warp_max(uint32_t v) { return __reduce_max_sync(FULL, v); }
// 64-bit sums (mod 2^64, so signed values too) as three REDUX sums of 22/21/21-bit slices: each slice
// sum over 32 lanes stays below 2^27, so the recombined total is exact; no shuffle chain (and no
// divergent-path copy of one)
__device__ __forceinline__ uint64_t warp_sum(uint64_t v) {
  const uint32_t lo = __reduce_add_sync(FULL, (uint32_t)v & 0x3fffffu);
  const uint32_t mi = __reduce_add_sync(FULL, (uint32_t)(v >> 22) & 0x1fffffu);
  const uint32_t hi = __reduce_add_sync(FULL, (uint32_t)(v >> 43));
  return (uint64_t)lo + ((uint64_t)mi << 22) + ((uint64_t)hi << 43);
}
__device__ __forceinline__ int64_t warp_sum(int64_t v) { return (int64_t)warp_sum((uint64_t)v); }
__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) { return warp_sum((uint64_t)v); }
__device__ __forceinline__ long long warp_sum(long long v) { return (long long)warp_sum((uint64_t)v); }
// inclusive scan across the warp
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int l = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T w = __shfl_up_sync(FULL, v, o);
    if (l >= o) v += w;
  }
  return v;
}

// ------------------------------------------------------------------ (key, idx) ordering ------
struct KI {
  int64_t k;
  int32_t i;
};
__device__ __forceinline__ bool ki_less(const KI& a, const KI& b) {
  return a.k < b.k || (a.k == b.k && a.i < b.i);
}
__device__ __forceinline__ KI ki_inf() { return KI{INF64, INF32}; }
__device__ __forceinline__ KI ki_shfl_xor(const KI& v, int m) {
  return KI{__shfl_xor_sync(FULL, v.k, m), __shfl_xor_sync(FULL, v.i, m)};
}
__device__ __forceinline__ KI ki_shfl(const KI& v, int src) {
  return KI{__shfl_sync(FULL, v.k, src), __shfl_sync(FULL, v.i, src)};
}
__device__ __forceinline__ KI ki_min(const KI& a, const KI& b) { return ki_less(b, a) ? b : a; }
__device__ __forceinline__ KI ki_max(const KI& a, const KI& b) { return ki_less(b, a) ? a : b; }

// Compare-exchange helpers: one (key, idx) comparison per exchange.
__device__ __forceinline__ KI ki_keep(const KI& v, const KI& o, bool keep_min) {
  const bool o_less = ki_less(o, v);
  return (o_less == keep_min) ? o : v;
}
__device__ __forceinline__ void ki_cas(KI& lo, KI& hi) {
  const bool sw = ki_less(hi, lo);
  const KI t = lo;
  lo = sw ? hi : lo;
  hi = sw ? t : hi;
}

// Bitonic sort of 32 elements, one per lane, ascending by lane.
__device__ __forceinline__ KI sort32(KI v) {
  const int l = lane_id();
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const KI o = ki_shfl_xor(v, j);
      const bool up = (l & k) == 0;
      const bool lower = (l & j) == 0;
      v = ki_keep(v, o, lower == up);
    }
  }
  return v;
}

// Warp-held sorted list of the K = 32*KPL smallest elements seen.
template <int KPL>
struct WarpTopK {
  KI a[KPL];

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int r = 0; r < KPL; r++) a[r] = ki_inf();
  }
  // a is bitonic after the min-with-reversed step; sort it ascending.
  __device__ __forceinline__ void bitonic_merge() {
    const int l = lane_id();
#pragma unroll
    for (int j = KPL / 2; j > 0; j >>= 1) {     // cross-register stages (stride j*32)
#pragma unroll
      for (int r = 0; r < KPL; r++) {
        if ((r & j) == 0) ki_cas(a[r], a[r | j]);
      }
    }
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {          // in-register stages across lanes
      const bool lower = (l & j) == 0;
#pragma unroll
      for (int r = 0; r < KPL; r++) {
        const KI o = ki_shfl_xor(a[r], j);
        a[r] = ki_keep(a[r], o, lower);
      }
    }
  }
  // merge a sorted 32-element warp vector b (one per lane, ascending) into the list
  __device__ __forceinline__ void merge32(const KI& b) {
    const KI br = ki_shfl(b, 31 - lane_id());
    a[KPL - 1] = ki_min(a[KPL - 1], br);
    bitonic_merge();
  }
  // merge another full sorted list (same layout)
  __device__ __forceinline__ void merge_list(const KI (&b)[KPL]) {
    const int src = 31 - lane_id();
#pragma unroll
    for (int r = 0; r < KPL; r++) a[r] = ki_min(a[r], ki_shfl(b[KPL - 1 - r], src));
    bitonic_merge();
  }
  __device__ __forceinline__ KI kth() const {  // current K-th smallest (the threshold)
    return ki_shfl(a[KPL - 1], 31);
  }
  // element at sorted position pos (0 <= pos < 32*KPL), broadcast to every lane
  __device__ __forceinline__ KI at(int pos) const {
    const int r = pos >> 5;
    KI x = a[0];
#pragma unroll
    for (int q = 1; q < KPL; q++) if (q == r) x = a[q];
    return ki_shfl(x, pos & 31);
  }
};

// Streaming front-end: candidates below the threshold are appended to a shared buffer (64 slots for
// push(); 160 for append() x4 + drain()) and
// merged 32 at a time, so a merge costs one sort32 + one bitonic merge per 32 survivors.  The
// threshold is the element at sorted position kpos (the last position the consumer can use:
// Algorithm 1 admits at most min(R, N-1, M-1, C-1) entries); kpos < 0 disables selection.
template <int KPL>
struct TopKStream {
  WarpTopK<KPL> top;
  KI thr;
  int cnt, kpos;
  bool any;  // has a merge happened (list non-empty)?
  KI* buf;   // 64 slots in shared memory (per warp)

  __device__ __forceinline__ void init(KI* sbuf, int kpos_ = 32 * KPL - 1) {
    top.init();
    thr = ki_inf();
    cnt = 0;
    kpos = kpos_;
    any = false;
    buf = sbuf;
  }
  __device__ __forceinline__ void flush32() {
    __syncwarp();
    KI y = buf[lane_id()];
    __syncwarp();
    for (int c0 = 32; c0 < cnt; c0 += 32) {  // shift the remaining candidates down by 32
      const int j = c0 + lane_id();
      KI rest = j < cnt ? buf[j] : ki_inf();
      __syncwarp();
      if (j < cnt) buf[j - 32] = rest;
      __syncwarp();
    }
    cnt -= 32;
    y = sort32(y);
    if (any) {
      top.merge32(y);
    } else {
      top.a[0] = y;  // first batch: the list was empty
      any = true;
    }
    thr = top.at(kpos);
    __syncwarp();
  }
  // offer one element per lane (valid = participates)
  __device__ __forceinline__ void push(const KI& x, bool valid) {
    const bool c = valid && ki_less(x, thr);
    const uint32_t m = __ballot_sync(FULL, c);
    if (m == 0) return;
    if (c) buf[cnt + __popc(m & lanemask_lt())] = x;
    cnt += __popc(m);
    if (cnt >= 32) flush32();
  }
  // append without merging (the buffer must hold cnt + 32): call drain() once per few pushes so
  // the merge network is instantiated at a single code location
  // c: this lane offers x (the caller already tested it against thr)
  __device__ __forceinline__ void append(const KI& x, bool c) {
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
      KI y = lane_id() < cnt ? buf[lane_id()] : ki_inf();
      __syncwarp();
      cnt = 0;
      y = sort32(y);
      if (any) top.merge32(y); else top.a[0] = y;
      any = true;
      thr = top.at(kpos);
    }
  }
};

// ------------------------------------------------------------- packed (key, idx) variant -------
// A (key, idx) pair whose key fits 32 bits relative to a base packs into one uint64 whose unsigned
// order is the (key, idx) order: ((key32 + 2^31) << 32) | idx32.  Compare-exchanges then cost one
// 64-bit compare and two shuffles instead of three.
constexpr uint64_t PK_INF = ~0ull;

__device__ __forceinline__ uint64_t pk_keep(uint64_t v, uint64_t o, bool keep_min) {
  return ((o < v) == keep_min) ? o : v;
}

__device__ __forceinline__ uint32_t sort32_u32(uint32_t v) {  // ascending by lane
  const int l = lane_id();
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint32_t o = __shfl_xor_sync(FULL, v, j);
      const bool keep_min = ((l & j) == 0) == ((l & k) == 0);
      v = ((o < v) == keep_min) ? o : v;
    }
  }
  return v;
}

__device__ __forceinline__ uint64_t sort32_pk(uint64_t v) {
  const int l = lane_id();
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint64_t o = __shfl_xor_sync(FULL, v, j);
      v = pk_keep(v, o, ((l & j) == 0) == ((l & k) == 0));
    }
  }
  return v;
}

}  // namespace asc
