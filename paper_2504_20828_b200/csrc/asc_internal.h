// asc_internal.h — context, workspace and kernel-launch declarations behind include/asc.h.
#pragma once
#include <cuda_runtime.h>

#include <string>

#include "../../include/asc.h"
#include "asc_dev.cuh"

constexpr int32_t ASC_PF_FAST_N = 1 << 17;  // entries of asc_ctx::d_pf_fast

struct asc_ctx {
  asc_config cfg;          // as given (tp not yet applied)
  int device = 0;
  int sms = 148;           // multiprocessors of `device` (queried once in asc_create)
  cudaStream_t stream = nullptr;
  asc::Model md;           // tp-divided model constants
  int32_t pt_size = 0;     // prefill table covers eff_prompt in [0, pt_size)
  int64_t* d_pf_tab = nullptr;  // prefill_us by eff_prompt (a1, cached per ctx)
  int32_t* d_pf_tab32 = nullptr;  // int32 copy for lookups (nullptr if some entry > INT32_MAX)
  int32_t* d_pf_tab32_mem = nullptr;
  int32_t* d_pf_fast = nullptr;  // [2^17]: prefill_us(q + 1), clipped to 2^30 (k1's fast path)
  int64_t w_hp = 0;        // worst-case HP batch latency (G24)
  int* d_err = nullptr;    // device error bits (asc::ERR_*)
  int* h_err = nullptr;    // mapped pinned host copy of the error bits (one sync per call)
  int* h_err_dev = nullptr;  // its device alias (err_publish writes it)
  char* ws = nullptr;      // device workspace
  size_t ws_cap = 0;
  char* stage = nullptr;   // device staging for host-pointer calls
  size_t stage_cap = 0;
  std::string err;
  int64_t last_kernel_launches = 0;  // kernels launched by the last call (bench evidence)
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;  // bracket the dominant kernel of the last call
  cudaEvent_t ev2 = nullptr, ev3 = nullptr;  // bracket its secondary kernel (schedule_step: k_lane)
  bool timed = false, timed2 = false;
  asc_snapshots snap{};     // armed decision snapshots for the next asc_simulate_batch
  bool snap_armed = false;
};

namespace asc {

// Host-side phase timer (experiments: ASC_HOST_PROF=1 prints the mean time per phase of
// asc_schedule_step at asc_destroy).  Off: one branch per mark.
struct HostProf {
  bool on = false;
  double acc[12] = {};
  long calls = 0;
  double last = 0;
  void mark(int i);
};
extern thread_local HostProf g_prof;  // per host thread (calls on one ctx come from one thread)

// bump allocator over a device buffer
struct Arena {
  char* base;
  size_t cap, off = 0;
  template <typename T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base + off);
    off += n * sizeof(T);
    return p;
  }
};

struct StepArgs;  // defined in step.cu
asc_status launch_schedule_step(asc_ctx* c, const asc_step_in* in, asc_step_out* out, int64_t Q);
asc_status launch_simulate(asc_ctx* c, const asc_traces* tr, asc_outcomes* out, int64_t R);
asc_status launch_goodput(asc_ctx* c, const asc_traces* tr, const asc_outcomes* out,
                          uint64_t* good, uint64_t* total);
asc_status launch_summary(asc_ctx* c, const asc_traces* tr, const asc_outcomes* out,
                          asc_summary* s);
asc_status launch_fit(asc_ctx* c, const asc_fit_in* in, int64_t N, double lambda, double* coef,
                      double* mean_err, double* max_err);
asc_status launch_latency(asc_ctx* c, int64_t n, const uint64_t* F, const uint64_t* M, int64_t* lat,
                          double* ts);
asc_status ensure_ws(asc_ctx* c, size_t bytes);
asc_status fail(asc_ctx* c, asc_status s, const std::string& msg);
asc_status cuda_check(asc_ctx* c, cudaError_t e, const char* what);
// read device error bits, reset them, map to a status
asc_status collect_errors(asc_ctx* c, const char* where);

}  // namespace asc
