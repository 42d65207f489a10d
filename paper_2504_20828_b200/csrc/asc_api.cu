#include <chrono>
// asc_api.cu — the C ABI of include/asc.h: validation, context, workspace, host staging.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "asc_internal.h"

using namespace asc;

static thread_local std::string g_create_err;

namespace asc {

thread_local HostProf g_prof;

__global__ void err_publish(int* d_err, int* h_err) {
  *h_err = *d_err;
  *d_err = 0;
}
static double now_us_host() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
void HostProf::mark(int i) {
  if (!on) return;
  const double t = now_us_host();
  if (i >= 0) acc[i] += t - last;
  last = t;
}

asc_status fail(asc_ctx* c, asc_status s, const std::string& msg) {
  if (c) c->err = msg; else g_create_err = msg;
  return s;
}

asc_status cuda_check(asc_ctx* c, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return ASC_OK;
  return fail(c, ASC_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

asc_status ensure_ws(asc_ctx* c, size_t bytes) {
  if (bytes <= c->ws_cap) return ASC_OK;
  if (c->ws) cudaFree(c->ws);
  c->ws = nullptr;
  c->ws_cap = 0;
  size_t cap = bytes + bytes / 8;
  if (cudaMalloc(&c->ws, cap) != cudaSuccess) {
    cudaGetLastError();
    return fail(c, ASC_E_NOMEM, "workspace allocation of " + std::to_string(cap) + " bytes failed");
  }
  c->ws_cap = cap;
  return ASC_OK;
}

static asc_status ensure_stage(asc_ctx* c, size_t bytes) {
  if (bytes <= c->stage_cap) return ASC_OK;
  if (c->stage) cudaFree(c->stage);
  c->stage = nullptr;
  c->stage_cap = 0;
  if (cudaMalloc(&c->stage, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(c, ASC_E_NOMEM, "staging allocation failed");
  }
  c->stage_cap = bytes;
  return ASC_OK;
}

asc_status collect_errors(asc_ctx* c, const char* where) {
  // one tiny kernel moves the bits to mapped pinned memory and clears them (instead of a D2H
  // copy plus a memset: one stream operation fewer on every call's critical path)
  err_publish<<<1, 1, 0, c->stream>>>(c->d_err, c->h_err_dev);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_check(c, e, where);
  const int bits = *(volatile int*)c->h_err;
  if (!bits) return ASC_OK;
  std::string w(where);
  if (bits & 8) return fail(c, ASC_E_CONFIG, w + ": request violates liveness validation (prompt_len, output_len >= 1; prompt+output <= lp_token_budget; ceil((prompt+output)/block_tokens) < kv_blocks), or a per-trace topology is out of range");
  if (bits & ERR_INVAL) return fail(c, ASC_E_INVAL, w + ": invalid input (eff_prompt < 1, seg_off decreasing, arrivals not sorted within a trace, or a fit record with y <= 0)");
  if (bits & ERR_RANGE) return fail(c, ASC_E_RANGE, w + ": range (F or M >= 2^53, or budget_reqs > ASC_MAX_BATCH)");
  if (bits & 16) return fail(c, ASC_E_EMPTY, w + ": goodput over a trace with 0 requests, or a fit group with fewer than 20 records");
  if (bits & 32) return fail(c, ASC_E_RANGE, w + ": regularised normal equations not positive definite");
  if (bits & ERR_INVARIANT) return fail(c, ASC_E_INVARIANT, w + ": invariant violated (queue left non-empty with no pending event)");
  return fail(c, ASC_E_INVARIANT, w + ": unknown device error");
}

}  // namespace asc

// prefill latency table for eff_prompt in [0, n) and the worst-case HP batch latency W_hp
__global__ void build_tables(Model md, int64_t* tab, int32_t* tab32, int32_t n, int32_t hp_tok,
                             int64_t* w_hp, int* err) {
  for (int32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const int64_t v = p == 0 ? 0 : prefill_lat(md, (uint64_t)p);
    if (v < 0) atomicOr(err, ERR_RANGE);
    tab[p] = v < 0 ? INT32_MAX : v;
    if (v > INT32_MAX) atomicOr((int*)(w_hp + 1), 1);  // int32 copy unusable
    tab32[p] = (int32_t)(v < 0 ? INT32_MAX : (v > INT32_MAX ? INT32_MAX : v));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t v = prefill_lat(md, (uint64_t)hp_tok);
    if (v < 0) atomicOr(err, ERR_RANGE);
    *w_hp = v;
  }
}

// k1's fast-path table: prefill_us(q + 1) for q in [0, n), values >= 2^30 stored as 2^30 (the fast
// path tests bit 30 and hands such tasks to the exact 64-bit path)
__global__ void build_fast_table(Model md, int32_t* tab, int32_t n) {
  for (int32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const int64_t v = prefill_lat(md, (uint64_t)q + 1);
    tab[q] = (int32_t)(v < 0 || v >= (int64_t(1) << 30) ? (int64_t(1) << 30) : v);
  }
}

extern "C" {

int32_t asc_abi_version(void) { return ASC_ABI_VERSION; }

const char* asc_last_error(const asc_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_err.c_str();
}

asc_status asc_create(const asc_config* cfg, int device, void* cuda_stream, asc_ctx** out) {
  { const char* e = getenv("ASC_HOST_PROF"); g_prof.on = e && *e == '1'; }
  if (!cfg || !out) return fail(nullptr, ASC_E_INVAL, "asc_create: NULL argument");
  *out = nullptr;
  const asc_arch& a = cfg->arch;
  const asc_topology& t = cfg->topo;
  const asc_flags& f = cfg->flags;
#define CHK(cond, msg) \
  if (!(cond)) return fail(nullptr, ASC_E_CONFIG, std::string("asc_create: ") + msg)
  CHK(a.h > 0 && a.n > 0 && a.s > 0 && a.m > 0 && a.L > 0 && a.b > 0 && a.dtype_bytes > 0 && a.tp > 0 && a.n_kv > 0,
      "arch fields must be positive (h, n, s, n_kv, m, L, b, dtype_bytes, tp)");
  CHK((int64_t)a.h == (int64_t)a.n * a.s, "arch.h != arch.n * arch.s");
  CHK(a.h % a.tp == 0 && a.n % a.tp == 0 && a.m % a.tp == 0 && a.n_kv % a.tp == 0,
      "arch.tp must divide h, n, n_kv and m (P:662)");
  CHK(cfg->perf.F_H > 0 && cfg->perf.M_H > 0, "perf.F_H and perf.M_H must be > 0");
  CHK(t.n_lp >= 1, "topo.n_lp must be >= 1");
  CHK(t.n_hp >= 0, "topo.n_hp must be >= 0");
  CHK(t.n_lp + t.n_hp <= ASC_MAX_INSTANCES, "topo.n_lp + topo.n_hp exceeds ASC_MAX_INSTANCES");
  CHK(t.block_tokens >= 1 && t.block_tokens <= 512, "topo.block_tokens must be in [1, 512]");
  CHK(t.kv_blocks_lp >= 1 && (t.n_hp == 0 || t.kv_blocks_hp >= 1), "topo.kv_blocks must be >= 1");
  CHK(t.kv_blocks_lp < (1 << 22) && t.kv_blocks_hp < (1 << 22), "topo.kv_blocks must be < 2^22");
  CHK(t.lp_max_batch >= 1 && t.lp_max_batch <= ASC_MAX_BATCH, "topo.lp_max_batch must be in [1, ASC_MAX_BATCH]");
  CHK(t.lp_token_budget >= 1 && t.lp_token_budget < (1 << 24), "topo.lp_token_budget must be in [1, 2^24)");
  CHK(t.hp_token_budget >= 1 && t.hp_token_budget < (1 << 24), "topo.hp_token_budget must be in [1, 2^24)");
  CHK(f.policy >= 0 && f.policy <= 5, "flags.policy must be an asc_policy");
  CHK(f.offload_rule == 0 || f.offload_rule == 1, "flags.offload_rule must be 0 or 1");
  CHK(f.key_w[0] >= -1024 && f.key_w[0] <= 1024 && f.key_w[1] >= -1024 && f.key_w[1] <= 1024 &&
          f.key_w[2] >= -1024 && f.key_w[2] <= 1024,
      "flags.key_w must be in [-1024, 1024]");
  CHK(f.offload_margin_us >= 0 && f.offload_delay_us >= 0, "flags.offload_margin_us/offload_delay_us must be >= 0");
  CHK(f.hist_default_tokens >= 0, "flags.hist_default_tokens must be >= 0");
  CHK(f.scheduler == ASC_SCHED_ASCENDRA || f.scheduler == ASC_SCHED_VLLM || f.scheduler == ASC_SCHED_SARATHI,
      "flags.scheduler must be an asc_scheduler");
  CHK(f.scheduler != ASC_SCHED_SARATHI || (f.chunk_tokens >= 1 && f.chunk_tokens < (1 << 24)),
      "flags.chunk_tokens must be in [1, 2^24) for ASC_SCHED_SARATHI");
  CHK(f.scheduler == ASC_SCHED_ASCENDRA || t.n_hp == 0,
      "flags.scheduler: baseline schedulers run on homogeneous instances (topo.n_hp must be 0)");
#undef CHK
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(nullptr, ASC_E_CUDA, "asc_create: no CUDA device (libasc has no CPU fallback)");
  }
  if (device < 0 || device >= ndev) return fail(nullptr, ASC_E_INVAL, "asc_create: bad device ordinal");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(nullptr, ASC_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  asc_ctx* c = new asc_ctx();
  c->cfg = *cfg;
  c->device = device;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  c->stream = (cudaStream_t)cuda_stream;
  // tp division
  const uint64_t tp = (uint64_t)a.tp;
  const uint64_t h = a.h / tp, n = a.n / tp, m = a.m / tp;
  c->md.n = n;
  c->md.s = (uint64_t)a.s;
  c->md.L = (uint64_t)a.L;
  c->md.d = (uint64_t)a.dtype_bytes;
  c->md.b = (uint64_t)a.b;
  c->md.W = 4 * h * h + 2 * h * m;
  c->md.FT = 4 * h * h + 2 * h * m;
  c->md.MT = 8 * h + 2 * m;
  {
    const uint64_t L = (uint64_t)a.L, d = (uint64_t)a.dtype_bytes, s2 = 2 * (uint64_t)a.s;
    c->md.dF_bd = L * c->md.FT;
    c->md.dF_sl = L * n * s2;
    c->md.dM_0 = L * d * c->md.W;
    c->md.dM_bd = L * d * (c->md.MT + n * s2);
    c->md.dM_sl = L * d * n * s2;
  }
  c->md.c0 = cfg->perf.c[0]; c->md.c1 = cfg->perf.c[1]; c->md.c2 = cfg->perf.c[2];
  c->md.c3 = cfg->perf.c[3]; c->md.c4 = cfg->perf.c[4];
  c->md.FH = cfg->perf.F_H;
  c->md.MH = cfg->perf.M_H;
  int32_t pt = t.lp_token_budget > t.hp_token_budget ? t.lp_token_budget : t.hp_token_budget;
  c->pt_size = pt + 1;
  int64_t* d_w = nullptr;
  if (cudaMalloc(&c->d_err, sizeof(int)) != cudaSuccess ||
      cudaHostAlloc((void**)&c->h_err, sizeof(int), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&c->h_err_dev, c->h_err, 0) != cudaSuccess ||
      cudaMalloc(&c->d_pf_tab, sizeof(int64_t) * c->pt_size) != cudaSuccess ||
      cudaMalloc(&c->d_pf_tab32_mem, sizeof(int32_t) * c->pt_size) != cudaSuccess ||
      cudaMalloc(&c->d_pf_fast, sizeof(int32_t) * ASC_PF_FAST_N) != cudaSuccess ||
      cudaMalloc(&d_w, 2 * sizeof(int64_t)) != cudaSuccess) {
    cudaGetLastError();
    asc_destroy(c);
    if (d_w) cudaFree(d_w);
    return fail(nullptr, ASC_E_NOMEM, "asc_create: device allocation failed");
  }
  cudaEventCreate(&c->ev0);
  cudaEventCreate(&c->ev1);
  cudaEventCreate(&c->ev2);
  cudaEventCreate(&c->ev3);
  cudaMemsetAsync(c->d_err, 0, sizeof(int), c->stream);
  cudaMemsetAsync(d_w, 0, 2 * sizeof(int64_t), c->stream);
  build_tables<<<(c->pt_size + 255) / 256, 256, 0, c->stream>>>(
      c->md, c->d_pf_tab, c->d_pf_tab32_mem, c->pt_size, t.hp_token_budget, d_w, c->d_err);
  build_fast_table<<<ASC_PF_FAST_N / 256, 256, 0, c->stream>>>(c->md, c->d_pf_fast, ASC_PF_FAST_N);
  int64_t hw[2] = {0, 0};
  e = cudaMemcpyAsync(hw, d_w, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream);
  asc_status st = e != cudaSuccess ? cuda_check(c, e, "asc_create") : collect_errors(c, "asc_create tables");
  c->w_hp = hw[0];
  c->d_pf_tab32 = hw[1] ? nullptr : c->d_pf_tab32_mem;
  cudaFree(d_w);
  if (st) {
    g_create_err = c->err;
    asc_destroy(c);
    return st;
  }
  *out = c;
  return ASC_OK;
}

void asc_destroy(asc_ctx* ctx) {
  if (!ctx) return;
  if (g_prof.on && g_prof.calls) {
    static const char* nm[] = {"checks", "ws+params", "planner", "k1", "k_lane+k_small", "k2+k3", "errors+sync"};
    fprintf(stderr, "asc host profile over %ld asc_schedule_step calls (us/call):", g_prof.calls);
    for (int i = 0; i < 7; i++) fprintf(stderr, " %s %.1f", nm[i], g_prof.acc[i] / g_prof.calls);
    fprintf(stderr, "\n");
    g_prof = HostProf{true};
  }
  if (ctx->d_err) cudaFree(ctx->d_err);
  if (ctx->h_err) cudaFreeHost(ctx->h_err);
  if (ctx->d_pf_tab) cudaFree(ctx->d_pf_tab);
  if (ctx->d_pf_tab32_mem) cudaFree(ctx->d_pf_tab32_mem);
  if (ctx->d_pf_fast) cudaFree(ctx->d_pf_fast);
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->stage) cudaFree(ctx->stage);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->ev2) cudaEventDestroy(ctx->ev2);
  if (ctx->ev3) cudaEventDestroy(ctx->ev3);
  delete ctx;
}

}  // extern "C"

// ------------------------------------------------------------------ host/device pointer kinds --
static int ptr_kind(const void* p) {  // 1 device, 0 host, -1 null
  if (!p) return -1;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) ? 1 : 0;
}

static bool same_kind(int kind, std::initializer_list<const void*> ps) {
  for (const void* p : ps)
    if (p && ptr_kind(p) != kind) return false;
  return true;
}

// Copies host arrays into the staging buffer and back.  The same sequence of up()/out() calls
// runs twice: first on a dry Stager (no base, no copies) that only sums the 256-byte-aligned
// offsets, which sizes the staging buffer, then for real -- so the size can never disagree with
// what is staged.
struct Stager {
  asc_ctx* c;
  bool dry = false;
  std::vector<std::pair<void*, const void*>> downs;  // (host dst, dev src) sizes below
  std::vector<size_t> down_sizes;
  size_t off = 0;
  char* base = nullptr;
  template <typename T>
  T* up(const T* h, size_t n) {
    if (!h) return nullptr;
    off = (off + 255) & ~size_t(255);
    T* d = dry ? nullptr : reinterpret_cast<T*>(base + off);
    off += n * sizeof(T);
    if (n && !dry) cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, c->stream);
    return d;
  }
  template <typename T>
  T* out(T* h, size_t n) {
    if (!h) return nullptr;
    off = (off + 255) & ~size_t(255);
    T* d = dry ? nullptr : reinterpret_cast<T*>(base + off);
    off += n * sizeof(T);
    if (!dry) {
      downs.push_back({(void*)h, (const void*)d});
      down_sizes.push_back(n * sizeof(T));
    }
    return d;
  }
  cudaError_t download() {
    for (size_t i = 0; i < downs.size(); i++)
      if (down_sizes[i])
        cudaMemcpyAsync(downs[i].first, downs[i].second, down_sizes[i], cudaMemcpyDeviceToHost, c->stream);
    return cudaStreamSynchronize(c->stream);
  }
};

// Runs plan(sg) on a dry Stager to size the staging buffer, then on the real one.
template <typename Plan>
static asc_status stage_host(asc_ctx* c, Stager& sg, Plan plan) {
  Stager dry{c};
  dry.dry = true;
  plan(dry);
  asc_status st = ensure_stage(c, dry.off + 256);
  if (st) return st;
  sg.base = c->stage;
  plan(sg);
  return ASC_OK;
}

// Host-pointer epilogue: the outputs are copied back even when the device flagged an error (so
// documented error markers such as asc_latency's -1 reach the caller), then the status returns.
static asc_status finish_host(asc_ctx* c, Stager& sg, const char* where) {
  asc_status st = collect_errors(c, where);
  cudaError_t e = sg.download();
  if (st) return st;
  return cuda_check(c, e, where);
}

extern "C" {

asc_status asc_schedule_step(asc_ctx* c, const asc_step_in* in, asc_step_out* out) {
  g_prof.mark(-1);
  if (g_prof.on) g_prof.calls++;
  if (!c || !in || !out) return fail(c, ASC_E_INVAL, "asc_schedule_step: NULL argument");
  if (c->cfg.flags.policy == ASC_POLICY_WEIGHTED || c->cfg.flags.offload_rule != 0)
    return fail(c, ASC_E_CONFIG, "asc_schedule_step: ASC_POLICY_WEIGHTED and offload_rule 1 are asc_simulate_batch only");
  c->err.clear();
  c->timed = false;
  c->timed2 = false;
  if (in->S < 0) return fail(c, ASC_E_INVAL, "asc_schedule_step: S < 0");
  if (!in->seg_off || !in->now_us || !in->deadline_us || !in->eff_prompt || !in->flags ||
      !in->dec_count || !in->dec_ctx_sum || !in->tbt_slo_us || !in->budget_tokens ||
      !in->budget_blocks || !in->budget_reqs || !out->admit_idx || !out->admit_cnt ||
      !out->offload_idx || !out->offload_cnt || !out->drop_idx || !out->drop_cnt || !out->batch_lat_us)
    return fail(c, ASC_E_INVAL, "asc_schedule_step: NULL array");
  cudaSetDevice(c->device);
  const int kind = ptr_kind(in->seg_off);
  if (!same_kind(kind, {in->now_us, in->deadline_us, in->eff_prompt, in->flags, in->dec_count,
                        in->dec_ctx_sum, in->tbt_slo_us, in->budget_tokens, in->budget_blocks,
                        in->budget_reqs, out->admit_idx, out->admit_cnt, out->offload_idx,
                        out->offload_cnt, out->drop_idx, out->drop_cnt, out->batch_lat_us,
                        out->prefill_us}))
    return fail(c, ASC_E_INVAL, "asc_schedule_step: host and device pointers mixed");
  const int32_t S = in->S;
  int64_t Q = in->Q;
  if (kind == 1) {
    if (Q < 0) {
      cudaError_t e = cudaMemcpy(&Q, in->seg_off + S, sizeof(int64_t), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return cuda_check(c, e, "asc_schedule_step: read seg_off[S]");
    }
  } else {
    if (Q >= 0 && Q != in->seg_off[S]) return fail(c, ASC_E_INVAL, "asc_schedule_step: Q != seg_off[S]");
    Q = in->seg_off[S];
    for (int32_t s = 0; s < S; s++)
      if (in->seg_off[s + 1] < in->seg_off[s]) return fail(c, ASC_E_INVAL, "asc_schedule_step: seg_off decreasing");
  }
  if (Q < 0) return fail(c, ASC_E_INVAL, "asc_schedule_step: seg_off[S] < 0");
  if (Q >= INT32_MAX) return fail(c, ASC_E_RANGE, "asc_schedule_step: total entries >= 2^31");
  asc_status st;
  if (kind == 1) {
    g_prof.mark(0);  // argument checks and pointer kinds
    st = launch_schedule_step(c, in, out, Q);
    if (st) return st;
    st = collect_errors(c, "asc_schedule_step");
    g_prof.mark(6);  // error read-back and stream sync
    return st;
  }
  const size_t Sn = (size_t)S, Qn = (size_t)Q;
  Stager sg{c};
  asc_step_in di = *in;
  asc_step_out dout;
  st = stage_host(c, sg, [&](Stager& sg) {
  di.seg_off = sg.up(in->seg_off, Sn + 1);
  di.now_us = sg.up(in->now_us, Sn);
  di.deadline_us = sg.up(in->deadline_us, Qn);
  di.eff_prompt = sg.up(in->eff_prompt, Qn);
  di.flags = sg.up(in->flags, Qn);
  di.dec_count = sg.up(in->dec_count, Sn);
  di.dec_ctx_sum = sg.up(in->dec_ctx_sum, Sn);
  di.tbt_slo_us = sg.up(in->tbt_slo_us, Sn);
  di.budget_tokens = sg.up(in->budget_tokens, Sn);
  di.budget_blocks = sg.up(in->budget_blocks, Sn);
  di.budget_reqs = sg.up(in->budget_reqs, Sn);
  dout.admit_idx = sg.out(out->admit_idx, Qn);
  dout.admit_cnt = sg.out(out->admit_cnt, Sn);
  dout.offload_idx = sg.out(out->offload_idx, Qn);
  dout.offload_cnt = sg.out(out->offload_cnt, Sn);
  dout.drop_idx = sg.out(out->drop_idx, Qn);
  dout.drop_cnt = sg.out(out->drop_cnt, Sn);
  dout.batch_lat_us = sg.out(out->batch_lat_us, Sn);
  dout.prefill_us = sg.out(out->prefill_us, Qn);
  });
  if (st) return st;
  st = launch_schedule_step(c, &di, &dout, Q);
  if (st) return st;
  return finish_host(c, sg, "asc_schedule_step");
}

asc_status asc_simulate_batch(asc_ctx* c, const asc_traces* tr, asc_outcomes* out) {
  if (!c || !tr || !out) return fail(c, ASC_E_INVAL, "asc_simulate_batch: NULL argument");
  c->err.clear();
  c->timed = false;
  c->timed2 = false;
  if (tr->T < 0) return fail(c, ASC_E_INVAL, "asc_simulate_batch: T < 0");
  if (!tr->trace_off || !tr->arrival_us || !tr->prompt_len || !tr->output_len || !tr->ttft_slo_us ||
      !tr->tbt_slo_us || !out->first_token_us || !out->done_us || !out->prefill_start_us ||
      !out->status || !out->digest)
    return fail(c, ASC_E_INVAL, "asc_simulate_batch: NULL array");
  cudaSetDevice(c->device);
  const int kind = ptr_kind(tr->trace_off);
  if (!same_kind(kind, {tr->arrival_us, tr->prompt_len, tr->output_len, tr->ttft_slo_us,
                        tr->tbt_slo_us, tr->req_ttft_slo_us, tr->n_lp, tr->n_hp, tr->req_key_offset_us,
                        out->first_token_us, out->done_us, out->prefill_start_us, out->status,
                        out->digest, out->decisions, out->evaluations}))
    return fail(c, ASC_E_INVAL, "asc_simulate_batch: host and device pointers mixed");
  const int32_t T = tr->T;
  int64_t R = tr->R;
  if (kind == 1) {
    if (R < 0) {
      cudaError_t e = cudaMemcpy(&R, tr->trace_off + T, sizeof(int64_t), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return cuda_check(c, e, "asc_simulate_batch: read trace_off[T]");
    }
  } else {
    if (R >= 0 && R != tr->trace_off[T]) return fail(c, ASC_E_INVAL, "asc_simulate_batch: R != trace_off[T]");
    R = tr->trace_off[T];
    for (int32_t t = 0; t < T; t++)
      if (tr->trace_off[t + 1] < tr->trace_off[t]) return fail(c, ASC_E_INVAL, "asc_simulate_batch: trace_off decreasing");
  }
  if (R < 0) return fail(c, ASC_E_INVAL, "asc_simulate_batch: trace_off[T] < 0");
  if (R >= INT32_MAX) return fail(c, ASC_E_RANGE, "asc_simulate_batch: total requests >= 2^31");
  asc_status st;
  if (kind == 1) {
    st = launch_simulate(c, tr, out, R);
    if (st) return st;
    return collect_errors(c, "asc_simulate_batch");
  }
  const size_t Tn = (size_t)T, Rn = (size_t)R;
  Stager sg{c};
  asc_traces dt = *tr;
  asc_outcomes doc = *out;
  st = stage_host(c, sg, [&](Stager& sg) {
  dt.trace_off = sg.up(tr->trace_off, Tn + 1);
  dt.arrival_us = sg.up(tr->arrival_us, Rn);
  dt.prompt_len = sg.up(tr->prompt_len, Rn);
  dt.output_len = sg.up(tr->output_len, Rn);
  dt.ttft_slo_us = sg.up(tr->ttft_slo_us, Tn);
  dt.tbt_slo_us = sg.up(tr->tbt_slo_us, Tn);
  dt.req_ttft_slo_us = sg.up(tr->req_ttft_slo_us, Rn);
  dt.n_lp = sg.up(tr->n_lp, Tn);
  dt.n_hp = sg.up(tr->n_hp, Tn);
  dt.req_key_offset_us = sg.up(tr->req_key_offset_us, Rn);
  doc.first_token_us = sg.out(out->first_token_us, Rn);
  doc.done_us = sg.out(out->done_us, Rn);
  doc.prefill_start_us = sg.out(out->prefill_start_us, Rn);
  doc.status = sg.out(out->status, Rn);
  doc.digest = sg.out(out->digest, Tn);
  doc.decisions = sg.out(out->decisions, Tn);
  doc.evaluations = sg.out(out->evaluations, Tn);
  });
  if (st) return st;
  st = launch_simulate(c, &dt, &doc, R);
  if (st) return st;
  return finish_host(c, sg, "asc_simulate_batch");
}

asc_status asc_goodput(asc_ctx* c, const asc_traces* tr, const asc_outcomes* out, uint64_t* good,
                       uint64_t* total) {
  if (!c || !tr || !out || !good || !total) return fail(c, ASC_E_INVAL, "asc_goodput: NULL argument");
  c->err.clear();
  c->timed = false;
  c->timed2 = false;
  if (tr->T < 0) return fail(c, ASC_E_INVAL, "asc_goodput: T < 0");
  cudaSetDevice(c->device);
  const int kind = ptr_kind(tr->trace_off);
  if (!same_kind(kind, {tr->arrival_us, tr->output_len, tr->ttft_slo_us, tr->tbt_slo_us,
                        tr->req_ttft_slo_us, out->first_token_us, out->done_us, out->status,
                        good, total}))
    return fail(c, ASC_E_INVAL, "asc_goodput: host and device pointers mixed");
  const int32_t T = tr->T;
  asc_status st;
  if (kind == 1) {
    st = launch_goodput(c, tr, out, good, total);
    if (st) return st;
    return collect_errors(c, "asc_goodput");
  }
  const size_t Tn = (size_t)T, Rn = (size_t)tr->trace_off[T];
  Stager sg{c};
  asc_traces dt = *tr;
  asc_outcomes doc{};
  uint64_t *dg = nullptr, *dtt = nullptr;
  st = stage_host(c, sg, [&](Stager& sg) {
  dt.trace_off = sg.up(tr->trace_off, Tn + 1);
  dt.arrival_us = sg.up(tr->arrival_us, Rn);
  dt.prompt_len = nullptr;
  dt.output_len = sg.up(tr->output_len, Rn);
  dt.ttft_slo_us = sg.up(tr->ttft_slo_us, Tn);
  dt.tbt_slo_us = sg.up(tr->tbt_slo_us, Tn);
  dt.req_ttft_slo_us = sg.up(tr->req_ttft_slo_us, Rn);
  doc.first_token_us = sg.up(out->first_token_us, Rn);
  doc.done_us = sg.up(out->done_us, Rn);
  doc.status = sg.up(out->status, Rn);
  dg = sg.out(good, Tn);
  dtt = sg.out(total, Tn);
  });
  if (st) return st;
  st = launch_goodput(c, &dt, &doc, dg, dtt);
  if (st) return st;
  return finish_host(c, sg, "asc_goodput");
}

asc_status asc_summarize(asc_ctx* c, const asc_traces* tr, const asc_outcomes* out, asc_summary* sum) {
  if (!c || !tr || !out || !sum) return fail(c, ASC_E_INVAL, "asc_summarize: NULL argument");
  c->err.clear();
  c->timed = false;
  c->timed2 = false;
  if (tr->T < 0) return fail(c, ASC_E_INVAL, "asc_summarize: T < 0");
  if (!tr->trace_off || !tr->arrival_us || !tr->output_len || !tr->ttft_slo_us || !tr->tbt_slo_us ||
      !out->first_token_us || !out->done_us || !out->prefill_start_us || !out->status)
    return fail(c, ASC_E_INVAL, "asc_summarize: NULL array");
  cudaSetDevice(c->device);
  const int kind = ptr_kind(tr->trace_off);
  int64_t** outs[] = {&sum->completed, &sum->dropped, &sum->violating, &sum->tokens,
                      &sum->ttft_p50_us, &sum->ttft_p90_us, &sum->ttft_p99_us, &sum->tbt_sum_us,
                      &sum->tbt_tokens, &sum->delay_sum_lp_us, &sum->delay_cnt_lp,
                      &sum->delay_sum_hp_us, &sum->delay_cnt_hp, &sum->last_done_us};
  if (!same_kind(kind, {tr->arrival_us, tr->output_len, tr->ttft_slo_us, tr->tbt_slo_us,
                        tr->req_ttft_slo_us, tr->n_lp, out->first_token_us, out->done_us,
                        out->prefill_start_us, out->status}))
    return fail(c, ASC_E_INVAL, "asc_summarize: host and device pointers mixed");
  for (int64_t** o : outs)
    if (!same_kind(kind, {*o})) return fail(c, ASC_E_INVAL, "asc_summarize: host and device pointers mixed");
  asc_status st;
  if (kind == 1) {
    st = launch_summary(c, tr, out, sum);
    if (st) return st;
    return collect_errors(c, "asc_summarize");
  }
  const int32_t T = tr->T;
  const size_t Tn = (size_t)T, Rn = (size_t)tr->trace_off[T];
  Stager sg{c};
  asc_traces dt = *tr;
  asc_outcomes doc{};
  asc_summary ds{};
  st = stage_host(c, sg, [&](Stager& sg) {
    dt.trace_off = sg.up(tr->trace_off, Tn + 1);
    dt.arrival_us = sg.up(tr->arrival_us, Rn);
    dt.prompt_len = nullptr;
    dt.output_len = sg.up(tr->output_len, Rn);
    dt.ttft_slo_us = sg.up(tr->ttft_slo_us, Tn);
    dt.tbt_slo_us = sg.up(tr->tbt_slo_us, Tn);
    dt.req_ttft_slo_us = sg.up(tr->req_ttft_slo_us, Rn);
    dt.n_lp = sg.up(tr->n_lp, Tn);
    dt.n_hp = nullptr;
    dt.req_key_offset_us = nullptr;
    doc.first_token_us = sg.up(out->first_token_us, Rn);
    doc.done_us = sg.up(out->done_us, Rn);
    doc.prefill_start_us = sg.up(out->prefill_start_us, Rn);
    doc.status = sg.up(out->status, Rn);
    int64_t** douts[] = {&ds.completed, &ds.dropped, &ds.violating, &ds.tokens, &ds.ttft_p50_us,
                         &ds.ttft_p90_us, &ds.ttft_p99_us, &ds.tbt_sum_us, &ds.tbt_tokens,
                         &ds.delay_sum_lp_us, &ds.delay_cnt_lp, &ds.delay_sum_hp_us,
                         &ds.delay_cnt_hp, &ds.last_done_us};
    for (int k = 0; k < 14; k++) *douts[k] = sg.out(*outs[k], Tn);
  });
  if (st) return st;
  st = launch_summary(c, &dt, &doc, &ds);
  if (st) return st;
  return finish_host(c, sg, "asc_summarize");
}

asc_status asc_fit_perf(asc_ctx* c, const asc_fit_in* in, double lambda, double* coef,
                        double* mean_err, double* max_err) {
  if (!c || !in || !coef) return fail(c, ASC_E_INVAL, "asc_fit_perf: NULL argument");
  c->err.clear();
  c->timed = false;
  c->timed2 = false;
  if (in->G < 0) return fail(c, ASC_E_INVAL, "asc_fit_perf: G < 0");
  if (!(lambda >= 0.0 && lambda < HUGE_VAL)) return fail(c, ASC_E_INVAL, "asc_fit_perf: lambda must be finite and >= 0");
  if (!in->rec_off || !in->F || !in->M || !in->y) return fail(c, ASC_E_INVAL, "asc_fit_perf: NULL array");
  cudaSetDevice(c->device);
  const int kind = ptr_kind(in->rec_off);
  if (!same_kind(kind, {in->F, in->M, in->y, coef, mean_err, max_err}))
    return fail(c, ASC_E_INVAL, "asc_fit_perf: host and device pointers mixed");
  const int32_t G = in->G;
  int64_t N = in->N;
  if (kind == 1) {
    if (N < 0) {
      cudaError_t e = cudaMemcpy(&N, in->rec_off + G, sizeof(int64_t), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return cuda_check(c, e, "asc_fit_perf: read rec_off[G]");
    }
    if (N < 0) return fail(c, ASC_E_INVAL, "asc_fit_perf: rec_off[G] < 0");
    asc_status st = launch_fit(c, in, N, lambda, coef, mean_err, max_err);
    if (st) return st;
    return collect_errors(c, "asc_fit_perf");
  }
  if (N < 0) N = in->rec_off[G];
  if (N != in->rec_off[G] || N < 0) return fail(c, ASC_E_INVAL, "asc_fit_perf: N != rec_off[G]");
  const size_t Gn = (size_t)G, Nn = (size_t)N;
  Stager sg{c};
  asc_fit_in d = *in;
  d.N = N;
  double *dc = nullptr, *dme = nullptr, *dmx = nullptr;
  asc_status st = stage_host(c, sg, [&](Stager& sg) {
  d.rec_off = sg.up(in->rec_off, Gn + 1);
  d.F = sg.up(in->F, Nn);
  d.M = sg.up(in->M, Nn);
  d.y = sg.up(in->y, Nn);
  dc = sg.out(coef, 5 * Gn);
  dme = sg.out(mean_err, Gn);
  dmx = sg.out(max_err, Gn);
  });
  if (st) return st;
  st = launch_fit(c, &d, N, lambda, dc, dme, dmx);
  if (st) return st;
  return finish_host(c, sg, "asc_fit_perf");
}

asc_status asc_latency(asc_ctx* c, int64_t n, const uint64_t* F, const uint64_t* M, int64_t* lat_us,
                       double* t_s) {
  if (!c) return fail(c, ASC_E_INVAL, "asc_latency: NULL context");
  c->err.clear();
  c->timed = false;
  c->timed2 = false;
  if (n < 0) return fail(c, ASC_E_INVAL, "asc_latency: n < 0");
  if (n == 0) { c->last_kernel_launches = 0; return ASC_OK; }
  if (!F || !M || !lat_us) return fail(c, ASC_E_INVAL, "asc_latency: NULL array");
  cudaSetDevice(c->device);
  const int kind = ptr_kind(F);
  if (!same_kind(kind, {M, lat_us, t_s})) return fail(c, ASC_E_INVAL, "asc_latency: host and device pointers mixed");
  asc_status st;
  if (kind == 1) {
    st = launch_latency(c, n, F, M, lat_us, t_s);
    if (st) return st;
    return collect_errors(c, "asc_latency");
  }
  const size_t nn = (size_t)n;
  Stager sg{c};
  const uint64_t *dF = nullptr, *dM = nullptr;
  int64_t* dl = nullptr;
  double* dt = nullptr;
  st = stage_host(c, sg, [&](Stager& sg) {
    dF = sg.up(F, nn);
    dM = sg.up(M, nn);
    dl = sg.out(lat_us, nn);
    dt = sg.out(t_s, nn);
  });
  if (st) return st;
  st = launch_latency(c, n, dF, dM, dl, dt);
  if (st) return st;
  return finish_host(c, sg, "asc_latency");
}

asc_status asc_arm_snapshots(asc_ctx* c, const asc_snapshots* s) {
  if (!c || !s) return fail(c, ASC_E_INVAL, "asc_arm_snapshots: NULL argument");
  if (s->every < 1 || s->max_snaps < 0 || s->entry_cap < 0 || s->out_cap < 0 || s->instance < 0 ||
      s->trace < 0 || !s->hdr || !s->counts || !s->ids || !s->deadline_us || !s->eff_prompt || !s->flags ||
      !s->out_ids)
    return fail(c, ASC_E_INVAL, "asc_arm_snapshots: bad argument");
  if (ptr_kind(s->hdr) != 1 || ptr_kind(s->counts) != 1 || ptr_kind(s->ids) != 1 || ptr_kind(s->out_ids) != 1 ||
      ptr_kind(s->deadline_us) != 1 || ptr_kind(s->eff_prompt) != 1 || ptr_kind(s->flags) != 1)
    return fail(c, ASC_E_INVAL, "asc_arm_snapshots: device pointers only");
  c->snap = *s;
  c->snap_armed = true;
  return ASC_OK;
}

int64_t asc_last_kernel_launches(const asc_ctx* c) { return c ? c->last_kernel_launches : 0; }

double asc_last_kernel_ms(const asc_ctx* c) {
  if (!c || !c->timed) return -1.0;
  float ms = -1.0f;
  if (cudaEventElapsedTime(&ms, c->ev0, c->ev1) != cudaSuccess) { cudaGetLastError(); return -1.0; }
  return (double)ms;
}

double asc_last_kernel2_ms(const asc_ctx* c) {
  if (!c || !c->timed2) return -1.0;
  float ms = -1.0f;
  if (cudaEventElapsedTime(&ms, c->ev2, c->ev3) != cudaSuccess) { cudaGetLastError(); return -1.0; }
  return (double)ms;
}

}  // extern "C"
