// fit.cu — asc_fit_perf: batched Eq. 4-5 calibration.
//
// For G independent groups of batch records (exact F flops, M bytes, observed seconds y) the
// ridge least-squares coefficients of t = C1 (tM+tF) + C2 max(tM,tF) + C3 tM + C4 tF + C5
// (G49).  The records are one flat HBM stream, cut into fixed chunks of FCH records;
// chunk c and group g intersect in at most one segment, whose 13 sufficient statistics (sums of
// tM², tF², tM·tF, x², x·tM, x·tF, tM, tF, x, y, tM·y, tF·y, x·y with x = max(tM, tF); the
// 5x5 Gram matrix and X'y of the features (tM+tF, x, tM, tF, 1) are linear in them) go to
// slot c + g of a partials array — unique along
// the monotone (chunk, group) staircase, and contiguous per group, so each group folds its
// partials in a fixed order (deterministic results, no atomics).  A thread per group then adds
// lambda, factors the 5x5 system (Cholesky) and solves it.  An optional second stream computes
// the in-sample relative errors of the fitted model.  HBM-bound: 24 B per record per pass.
#include "asc_internal.h"

using namespace asc;

namespace {

constexpr int FCH = 8192;   // records per chunk
constexpr int FT = 256;     // threads per CTA
constexpr int NS = 13;      // sufficient statistics per segment (see acc1)
constexpr int ERR_FIT_SMALL = 16, ERR_FIT_PD = 32;

struct FitP {
  int32_t G;
  int32_t vec;     // F, M, y 16-byte aligned: 2-record vector loads
  int64_t N, nch;
  const int64_t* off;
  const uint64_t* F;
  const uint64_t* M;
  const double* y;
  double rMH, rFH, lam;  // 1 / M_H, 1 / F_H
  double* part;    // [(nch + G) * NS]
  double* part2;   // [(nch + G) * 2]: Σ relative error, max relative error
  double* coef;    // [G * 5]
  double* mean_err;
  double* max_err;
  int* err;
};

// largest g with off[g] <= r (off non-decreasing, off[0] = 0 <= r < off[G])
__device__ __forceinline__ int32_t group_of(const FitP& p, int64_t r) {
  int32_t lo = 0, hi = p.G;
  while (hi - lo > 1) {
    const int32_t mid = (lo + hi) >> 1;
    if (__ldg(p.off + mid) <= r) lo = mid; else hi = mid;
  }
  return lo;
}

// tM = M / M_H and tF = F / F_H as products with the reciprocals (within an ulp of the quotients)
__device__ __forceinline__ void times(const FitP& p, uint64_t F, uint64_t M, double& tM, double& tF) {
  tM = __dmul_rn(__ull2double_rn(M), p.rMH);
  tF = __dmul_rn(__ull2double_rn(F), p.rFH);
}

__device__ __forceinline__ void acc1(const FitP& p, double (&s)[NS], uint64_t F, uint64_t M, double y) {
  if (!(y > 0.0 && y < INFINITY)) atomicOr(p.err, ERR_INVAL);  // observed seconds > 0
  double tM, tF;
  times(p, F, M, tM, tF);
  const double x = tM > tF ? tM : tF;
  s[0] = __fma_rn(tM, tM, s[0]);
  s[1] = __fma_rn(tF, tF, s[1]);
  s[2] = __fma_rn(tM, tF, s[2]);
  s[3] = __fma_rn(x, x, s[3]);
  s[4] = __fma_rn(x, tM, s[4]);
  s[5] = __fma_rn(x, tF, s[5]);
  s[6] = __dadd_rn(s[6], tM);
  s[7] = __dadd_rn(s[7], tF);
  s[8] = __dadd_rn(s[8], x);
  s[9] = __dadd_rn(s[9], y);
  s[10] = __fma_rn(tM, y, s[10]);
  s[11] = __fma_rn(tF, y, s[11]);
  s[12] = __fma_rn(x, y, s[12]);
}

// block-wide sum of v[0..K) (fixed order: warp butterflies, then warps in index order)
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* sm, double* out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; k++) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] = __dadd_rn(v[k], __shfl_xor_sync(FULL, v[k], o));
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; k++) sm[w * K + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double s = 0.0;
    for (int j = 0; j < FT / 32; j++) s = __dadd_rn(s, sm[j * K + threadIdx.x]);
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// Per-thread sums over records [a, b) of one group: thread t takes records a + 2t, a + 2t + 1,
// then strides by 2 FT (16-byte loads of F, M and y when aligned), else one record per step.
template <class Body>
__device__ __forceinline__ void for_records(const FitP& p, int64_t a, int64_t b, Body body) {
  if (p.vec && ((a & 1) == 0)) {
    int64_t i = a + 2 * (int64_t)threadIdx.x;
#pragma unroll 2
    for (; i + 1 < b; i += 2 * FT) {
      const ulonglong2 f2 = __ldcs(reinterpret_cast<const ulonglong2*>(p.F + i));
      const ulonglong2 m2 = __ldcs(reinterpret_cast<const ulonglong2*>(p.M + i));
      const double2 y2 = __ldcs(reinterpret_cast<const double2*>(p.y + i));
      body(f2.x, m2.x, y2.x);
      body(f2.y, m2.y, y2.y);
    }
    if (i < b) body(__ldcs(p.F + i), __ldcs(p.M + i), __ldcs(p.y + i));  // odd tail
  } else {
#pragma unroll 4
    for (int64_t i = a + threadIdx.x; i < b; i += FT) body(__ldcs(p.F + i), __ldcs(p.M + i), __ldcs(p.y + i));
  }
}

__global__ void __launch_bounds__(FT, 4) fit_partials(const __grid_constant__ FitP p) {
  __shared__ double sm[(FT / 32) * NS];
  for (int64_t c = blockIdx.x; c < p.nch; c += gridDim.x) {
    const int64_t lo = c * FCH, hi = min(lo + FCH, p.N);
    for (int32_t g = group_of(p, lo); g < p.G; g++) {
      const int64_t a = max(__ldg(p.off + g), lo), b = min(__ldg(p.off + g + 1), hi);
      if (a < b) {
        double s[NS];
#pragma unroll
        for (int k = 0; k < NS; k++) s[k] = 0.0;
        for_records(p, a, b, [&](uint64_t F, uint64_t M, double y) { acc1(p, s, F, M, y); });
        block_sum<NS>(s, sm, p.part + (c + g) * NS);
      }
      if (__ldg(p.off + g + 1) >= hi) break;
    }
  }
}

// one thread per group: fold the group's segments in chunk order, + lambda, Cholesky, solve
__global__ void fit_solve(const __grid_constant__ FitP p) {
  const int32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= p.G) return;
  const int64_t lo = p.off[g], hi = p.off[g + 1];
  if (hi - lo < 20) { atomicOr(p.err, ERR_FIT_SMALL); return; }
  double s[NS];
  for (int k = 0; k < NS; k++) s[k] = 0.0;
  for (int64_t c = lo / FCH; c <= (hi - 1) / FCH; c++)
    for (int k = 0; k < NS; k++) s[k] = __dadd_rn(s[k], p.part[(c + g) * NS + k]);
  // Gram matrix and X'y of x = (tM + tF, m, tM, tF, 1), m = max(tM, tF), from the statistics
  const double mm = s[0], ff = s[1], mf = s[2], xx = s[3], xm = s[4], xf = s[5], sM = s[6],
               sF = s[7], sX = s[8], sy = s[9], my = s[10], fy = s[11], xy = s[12];
  const double n = (double)(hi - lo);
  double A[5][5], bb[5];
  A[0][0] = __dadd_rn(__dadd_rn(mm, __dmul_rn(2.0, mf)), ff);
  A[0][1] = __dadd_rn(xm, xf);
  A[0][2] = __dadd_rn(mm, mf);
  A[0][3] = __dadd_rn(mf, ff);
  A[0][4] = __dadd_rn(sM, sF);
  A[1][1] = xx; A[1][2] = xm; A[1][3] = xf; A[1][4] = sX;
  A[2][2] = mm; A[2][3] = mf; A[2][4] = sM;
  A[3][3] = ff; A[3][4] = sF;
  A[4][4] = n;
  for (int j = 0; j < 5; j++)
    for (int k = 0; k < j; k++) A[j][k] = A[k][j];
  bb[0] = __dadd_rn(my, fy); bb[1] = xy; bb[2] = my; bb[3] = fy; bb[4] = sy;
  for (int j = 0; j < 5; j++) A[j][j] = __dadd_rn(A[j][j], p.lam);
  double L[5][5];
  for (int j = 0; j < 5; j++) {
    double d = A[j][j];
    for (int k = 0; k < j; k++) d = __dsub_rn(d, __dmul_rn(L[j][k], L[j][k]));
    if (!(d > 0.0)) { atomicOr(p.err, ERR_FIT_PD); return; }
    L[j][j] = __dsqrt_rn(d);
    for (int i = j + 1; i < 5; i++) {
      double v = A[i][j];
      for (int k = 0; k < j; k++) v = __dsub_rn(v, __dmul_rn(L[i][k], L[j][k]));
      L[i][j] = __ddiv_rn(v, L[j][j]);
    }
  }
  double z[5], cc[5];
  for (int i = 0; i < 5; i++) {
    double v = bb[i];
    for (int k = 0; k < i; k++) v = __dsub_rn(v, __dmul_rn(L[i][k], z[k]));
    z[i] = __ddiv_rn(v, L[i][i]);
  }
  for (int i = 4; i >= 0; i--) {
    double v = z[i];
    for (int k = i + 1; k < 5; k++) v = __dsub_rn(v, __dmul_rn(L[k][i], cc[k]));
    cc[i] = __ddiv_rn(v, L[i][i]);
  }
  for (int j = 0; j < 5; j++) p.coef[5 * g + j] = cc[j];
}

// in-sample relative error of the fitted model (Eq. 4-5 prediction, clamped at 0)
__global__ void __launch_bounds__(FT, 4) fit_resid(const __grid_constant__ FitP p) {
  __shared__ double sm[(FT / 32) * 2];
  __shared__ double smx[FT / 32];
  for (int64_t c = blockIdx.x; c < p.nch; c += gridDim.x) {
    const int64_t lo = c * FCH, hi = min(lo + FCH, p.N);
    for (int32_t g = group_of(p, lo); g < p.G; g++) {
      const int64_t a = max(__ldg(p.off + g), lo), b = min(__ldg(p.off + g + 1), hi);
      if (a < b) {
        const double c0 = p.coef[5 * g], c1 = p.coef[5 * g + 1], c2 = p.coef[5 * g + 2],
                     c3 = p.coef[5 * g + 3], c4 = p.coef[5 * g + 4];
        double v[1] = {0.0}, mx = 0.0;
        for_records(p, a, b, [&](uint64_t F, uint64_t M, double yi) {
          double tM, tF;
          times(p, F, M, tM, tF);
          double t = __dmul_rn(c0, __dadd_rn(tM, tF));
          t = __dadd_rn(t, __dmul_rn(c1, tM > tF ? tM : tF));
          t = __dadd_rn(t, __dmul_rn(c2, tM));
          t = __dadd_rn(t, __dmul_rn(c3, tF));
          t = __dadd_rn(t, c4);
          if (!(t > 0.0)) t = 0.0;
          const double e = __ddiv_rn(fabs(__dsub_rn(t, yi)), yi);
          v[0] = __dadd_rn(v[0], e);
          mx = e > mx ? e : mx;
        });
        for (int o = 16; o > 0; o >>= 1) {
          const double m2 = __shfl_xor_sync(FULL, mx, o);
          mx = m2 > mx ? m2 : mx;
        }
        if ((threadIdx.x & 31) == 0) smx[threadIdx.x >> 5] = mx;
        block_sum<1>(v, sm, p.part2 + (c + g) * 2);  // (its syncs order the smx writes too)
        if (threadIdx.x == 0) {
          double m = 0.0;
          for (int j = 0; j < FT / 32; j++) m = smx[j] > m ? smx[j] : m;
          p.part2[(c + g) * 2 + 1] = m;
        }
        __syncthreads();
      }
      if (__ldg(p.off + g + 1) >= hi) break;
    }
  }
}

__global__ void fit_resid_final(const __grid_constant__ FitP p) {
  const int32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= p.G) return;
  const int64_t lo = p.off[g], hi = p.off[g + 1];
  if (hi - lo < 20) return;
  double s = 0.0, m = 0.0;
  for (int64_t c = lo / FCH; c <= (hi - 1) / FCH; c++) {
    s = __dadd_rn(s, p.part2[(c + g) * 2]);
    const double x = p.part2[(c + g) * 2 + 1];
    m = x > m ? x : m;
  }
  if (p.mean_err) p.mean_err[g] = __ddiv_rn(s, (double)(hi - lo));
  if (p.max_err) p.max_err[g] = m;
}

// asc_latency: Eq. 4-5 (+ G17/G18) per (F, M) pair, the same t_from_FM the schedulers use.  16 B in,
// 8 (+8) B out per pair; grid-stride over a resident grid.
__global__ void __launch_bounds__(256) latency_kernel(Model md, int64_t n, const uint64_t* __restrict__ F,
                                                      const uint64_t* __restrict__ M, int64_t* __restrict__ lat,
                                                      double* __restrict__ ts, int* err) {
  // LU pairs per thread per pass, all loads issued before the arithmetic (memory-level parallelism)
  constexpr int LU = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += LU * stride) {
    uint64_t f[LU], m[LU];
#pragma unroll
    for (int u = 0; u < LU; u++) {
      const int64_t i = i0 + u * stride;
      f[u] = i < n ? __ldcs(F + i) : 0;
      m[u] = i < n ? __ldcs(M + i) : 0;
    }
#pragma unroll
    for (int u = 0; u < LU; u++) {
      const int64_t i = i0 + u * stride;
      if (i >= n) break;
      if (f[u] >= TWO53 || m[u] >= TWO53) {  // int -> double would not be exact
        atomicOr(err, ERR_RANGE);
        lat[i] = -1;
        if (ts) ts[i] = 0.0;
        continue;
      }
      const double t = t_from_FM(md, f[u], m[u]);
      __stcs(lat + i, (long long)us_of_t(t));
      if (ts) __stcs(ts + i, t);
    }
  }
}

}  // namespace

namespace asc {

asc_status launch_latency(asc_ctx* c, int64_t n, const uint64_t* F, const uint64_t* M, int64_t* lat,
                          double* ts) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  int64_t grid = (n + 4 * 256 - 1) / (4 * 256);
  if (grid > (int64_t)sms * 8) grid = (int64_t)sms * 8;
  int64_t launches = 0;
  if (n > 0) {
    cudaEventRecord(c->ev0, c->stream);
    latency_kernel<<<(unsigned)grid, 256, 0, c->stream>>>(c->md, n, F, M, lat, ts, c->d_err);
    cudaEventRecord(c->ev1, c->stream);
    c->timed = true;
    launches++;
  }
  c->last_kernel_launches = launches;
  return cuda_check(c, cudaGetLastError(), "latency launch");
}

asc_status launch_fit(asc_ctx* c, const asc_fit_in* in, int64_t N, double lambda, double* coef,
                      double* mean_err, double* max_err) {
  FitP p{};
  p.G = in->G;
  p.N = N;
  p.nch = (N + FCH - 1) / FCH;
  p.off = in->rec_off;
  p.F = in->F;
  p.M = in->M;
  p.y = in->y;
  p.rMH = 1.0 / c->md.MH;
  p.rFH = 1.0 / c->md.FH;
  p.vec = ((reinterpret_cast<uintptr_t>(in->F) | reinterpret_cast<uintptr_t>(in->M) |
            reinterpret_cast<uintptr_t>(in->y)) & 15) == 0;
  p.lam = lambda;
  p.coef = coef;
  p.mean_err = mean_err;
  p.max_err = max_err;
  p.err = c->d_err;
  const bool resid = mean_err || max_err;
  const size_t nseg = (size_t)(p.nch + p.G);
  asc_status st = ensure_ws(c, nseg * NS * 8 + (resid ? nseg * 16 : 0) + 4096);
  if (st) return st;
  Arena ar{c->ws, c->ws_cap};
  p.part = ar.take<double>(nseg * NS);
  p.part2 = resid ? ar.take<double>(nseg * 2) : nullptr;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  int per_sm = 4;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fit_partials, FT, 0);
  int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  if (grid > p.nch) grid = p.nch;
  const unsigned gs = (unsigned)((p.G + 127) / 128);
  int64_t launches = 0;
  if (p.G > 0) {
    cudaEventRecord(c->ev0, c->stream);
    if (grid > 0) { fit_partials<<<(unsigned)grid, FT, 0, c->stream>>>(p); launches++; }
    cudaEventRecord(c->ev1, c->stream);
    c->timed = true;
    fit_solve<<<gs, 128, 0, c->stream>>>(p);
    launches++;
    if (resid) {
      if (grid > 0) { fit_resid<<<(unsigned)grid, FT, 0, c->stream>>>(p); launches++; }
      fit_resid_final<<<gs, 128, 0, c->stream>>>(p);
      launches++;
    }
  }
  c->last_kernel_launches = launches;
  return cuda_check(c, cudaGetLastError(), "fit launch");
}

}  // namespace asc
