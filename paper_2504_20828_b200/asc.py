"""Thin ctypes binding of include/asc.h (argument marshalling only).

Every step of the hot path runs in libasc.so's sm_100a kernels; this module only converts
preset dicts into asc_config, and torch CUDA tensors (device pointers) or numpy arrays (host
pointers, staged by the library itself) into the C structs.  There is no CPU fallback: if
libasc.so is missing or no CUDA device is present, the calls raise.
"""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ASC_LIB", os.path.join(_HERE, "libasc.so"))
_LIB = None

ASC_MAX_BATCH = 128
ASC_MAX_INSTANCES = 16
STATUS = {0: "ASC_OK", 1: "ASC_E_INVAL", 2: "ASC_E_CONFIG", 3: "ASC_E_NOMEM", 4: "ASC_E_CUDA",
          5: "ASC_E_EMPTY", 6: "ASC_E_RANGE", 7: "ASC_E_INVARIANT"}
EXPORTS = ("asc_create", "asc_destroy", "asc_last_error", "asc_abi_version", "asc_schedule_step",
           "asc_simulate_batch", "asc_goodput", "asc_summarize", "asc_fit_perf", "asc_latency", "asc_last_kernel_launches",
           "asc_last_kernel_ms", "asc_last_kernel2_ms", "asc_arm_snapshots")


class asc_snapshots(C.Structure):
    _fields_ = [("trace", C.c_int32), ("instance", C.c_int32), ("every", C.c_int64),
                ("max_snaps", C.c_int32), ("entry_cap", C.c_int64), ("out_cap", C.c_int64),
                ("hdr", C.c_void_p), ("counts", C.c_void_p), ("ids", C.c_void_p),
                ("deadline_us", C.c_void_p), ("eff_prompt", C.c_void_p), ("flags", C.c_void_p),
                ("out_ids", C.c_void_p)]


class AscError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class asc_arch(C.Structure):
    _fields_ = [(k, C.c_int32) for k in ("h", "n", "s", "n_kv", "m", "L", "b", "dtype_bytes", "tp")]


class asc_perf(C.Structure):
    _fields_ = [("c", C.c_double * 5), ("F_H", C.c_double), ("M_H", C.c_double)]


class asc_topology(C.Structure):
    _fields_ = [(k, C.c_int32) for k in ("n_lp", "n_hp", "block_tokens", "kv_blocks_lp",
                                         "kv_blocks_hp", "lp_max_batch", "lp_token_budget",
                                         "hp_token_budget")]


class asc_flags(C.Structure):
    _fields_ = [("policy", C.c_int32), ("offload", C.c_uint8), ("tickets", C.c_uint8),
                ("elastic", C.c_uint8), ("drop", C.c_uint8), ("offload_margin_us", C.c_int64),
                ("offload_delay_us", C.c_int64), ("hist_default_tokens", C.c_int32),
                ("scheduler", C.c_int32), ("chunk_tokens", C.c_int32),
                ("offload_rule", C.c_int32), ("key_w", C.c_int32 * 3)]


class asc_config(C.Structure):
    _fields_ = [("arch", asc_arch), ("perf", asc_perf), ("topo", asc_topology), ("flags", asc_flags)]


_P = C.c_void_p


class asc_step_in(C.Structure):
    _fields_ = [("S", C.c_int32), ("Q", C.c_int64)] + [(k, _P) for k in (
        "seg_off", "now_us", "deadline_us", "eff_prompt", "flags", "dec_count", "dec_ctx_sum",
        "tbt_slo_us", "budget_tokens", "budget_blocks", "budget_reqs")]


class asc_step_out(C.Structure):
    _fields_ = [(k, _P) for k in ("admit_idx", "admit_cnt", "offload_idx", "offload_cnt",
                                  "drop_idx", "drop_cnt", "batch_lat_us", "prefill_us")]


class asc_traces(C.Structure):
    _fields_ = [("T", C.c_int32), ("R", C.c_int64)] + [(k, _P) for k in (
        "trace_off", "arrival_us", "prompt_len", "output_len", "ttft_slo_us", "tbt_slo_us",
        "req_ttft_slo_us", "n_lp", "n_hp", "req_key_offset_us")]


class asc_fit_in(C.Structure):
    _fields_ = [("G", C.c_int32), ("N", C.c_int64)] + [(k, _P) for k in ("rec_off", "F", "M", "y")]


class asc_outcomes(C.Structure):
    _fields_ = [(k, _P) for k in ("first_token_us", "done_us", "prefill_start_us", "status",
                                  "digest", "decisions", "evaluations")]


SUMMARY_KEYS = ("completed", "dropped", "violating", "tokens", "ttft_p50_us", "ttft_p90_us",
                "ttft_p99_us", "tbt_sum_us", "tbt_tokens", "delay_sum_lp_us", "delay_cnt_lp",
                "delay_sum_hp_us", "delay_cnt_hp", "last_done_us")


class asc_summary(C.Structure):
    _fields_ = [(k, _P) for k in SUMMARY_KEYS]


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.asc_create.argtypes = [C.POINTER(asc_config), C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]
        L.asc_create.restype = C.c_int
        L.asc_destroy.argtypes = [C.c_void_p]
        L.asc_destroy.restype = None
        L.asc_last_error.argtypes = [C.c_void_p]
        L.asc_last_error.restype = C.c_char_p
        L.asc_abi_version.restype = C.c_int32
        L.asc_schedule_step.argtypes = [C.c_void_p, C.POINTER(asc_step_in), C.POINTER(asc_step_out)]
        L.asc_schedule_step.restype = C.c_int
        L.asc_simulate_batch.argtypes = [C.c_void_p, C.POINTER(asc_traces), C.POINTER(asc_outcomes)]
        L.asc_simulate_batch.restype = C.c_int
        L.asc_goodput.argtypes = [C.c_void_p, C.POINTER(asc_traces), C.POINTER(asc_outcomes),
                                  C.c_void_p, C.c_void_p]
        L.asc_goodput.restype = C.c_int
        L.asc_summarize.argtypes = [C.c_void_p, C.POINTER(asc_traces), C.POINTER(asc_outcomes),
                                    C.POINTER(asc_summary)]
        L.asc_summarize.restype = C.c_int
        L.asc_fit_perf.argtypes = [C.c_void_p, C.POINTER(asc_fit_in), C.c_double, C.c_void_p,
                                   C.c_void_p, C.c_void_p]
        L.asc_fit_perf.restype = C.c_int
        L.asc_latency.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.asc_latency.restype = C.c_int
        L.asc_last_kernel_launches.argtypes = [C.c_void_p]
        L.asc_last_kernel_launches.restype = C.c_int64
        L.asc_last_kernel_ms.argtypes = [C.c_void_p]
        L.asc_last_kernel_ms.restype = C.c_double
        L.asc_last_kernel2_ms.argtypes = [C.c_void_p]
        L.asc_last_kernel2_ms.restype = C.c_double
        L.asc_arm_snapshots.argtypes = [C.c_void_p, C.POINTER(asc_snapshots)]
        L.asc_arm_snapshots.restype = C.c_int
        _LIB = L
    return _LIB


def make_config(cfg):
    a, p, t, f = cfg["arch"], cfg["perf"], cfg["topo"], cfg["flags"]
    return asc_config(
        asc_arch(a["h"], a["n"], a["s"], a["n_kv"], a["m"], a["L"], a["b"], a["dtype_bytes"], a["tp"]),
        asc_perf((C.c_double * 5)(*p["c"]), p["F_H"], p["M_H"]),
        asc_topology(t["n_lp"], t["n_hp"], t["block_tokens"], t["kv_blocks_lp"], t["kv_blocks_hp"],
                     t["lp_max_batch"], t["lp_token_budget"], t["hp_token_budget"]),
        asc_flags(f["policy"], f["offload"], f["tickets"], f["elastic"], f["drop"],
                  f["offload_margin_us"], f["offload_delay_us"], f["hist_default_tokens"],
                  f.get("scheduler", 0), f.get("chunk_tokens", 512), f.get("offload_rule", 0),
                  (C.c_int32 * 3)(*f.get("key_weights", (1, -1, 0)))))


def _ptr(x):
    """Device pointer of a torch tensor, host pointer of a numpy array, or NULL."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return x.ctypes.data
    assert x.is_contiguous()
    return x.data_ptr()


def _check(ctx, rc, what):
    if rc != 0:
        msg = lib().asc_last_error(ctx)
        raise AscError(rc, f"{what}: {msg.decode() if msg else ''}")


def asc_create(cfg, device=0, stream=None):
    """Returns an opaque ctx handle (int).  stream: torch.cuda.Stream, raw handle or None."""
    h = C.c_void_p()
    sp = None
    if stream is not None:
        sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    c = make_config(cfg)
    rc = lib().asc_create(C.byref(c), int(device), sp, C.byref(h))
    _check(None, rc, "asc_create")
    return h.value


def asc_destroy(ctx):
    lib().asc_destroy(ctx)


def asc_last_kernel_launches(ctx):
    return int(lib().asc_last_kernel_launches(ctx))


def asc_last_kernel_ms(ctx):
    return float(lib().asc_last_kernel_ms(ctx))


def asc_last_kernel2_ms(ctx):
    return float(lib().asc_last_kernel2_ms(ctx))


def asc_schedule_step(ctx, seg_off, now_us, deadline_us, eff_prompt, flags, dec_count, dec_ctx_sum,
                      tbt_slo_us, budget_tokens, budget_blocks, budget_reqs, admit_idx, admit_cnt,
                      offload_idx, offload_cnt, drop_idx, drop_cnt, batch_lat_us, prefill_us=None,
                      Q=-1):
    S = len(seg_off) - 1
    i = asc_step_in(S, Q, *[_ptr(x) for x in (seg_off, now_us, deadline_us, eff_prompt, flags,
                                           dec_count, dec_ctx_sum, tbt_slo_us, budget_tokens,
                                           budget_blocks, budget_reqs)])
    o = asc_step_out(*[_ptr(x) for x in (admit_idx, admit_cnt, offload_idx, offload_cnt, drop_idx,
                                         drop_cnt, batch_lat_us, prefill_us)])
    _check(ctx, lib().asc_schedule_step(ctx, C.byref(i), C.byref(o)), "asc_schedule_step")


def asc_simulate_batch(ctx, trace_off, arrival_us, prompt_len, output_len, ttft_slo_us, tbt_slo_us,
                       first_token_us, done_us, prefill_start_us, status, digest, decisions=None,
                       evaluations=None, req_ttft_slo_us=None, R=-1, n_lp=None, n_hp=None,
                       req_key_offset_us=None):
    T = len(trace_off) - 1
    tr = asc_traces(T, R, *[_ptr(x) for x in (trace_off, arrival_us, prompt_len, output_len,
                                           ttft_slo_us, tbt_slo_us, req_ttft_slo_us, n_lp, n_hp,
                                           req_key_offset_us)])
    oc = asc_outcomes(*[_ptr(x) for x in (first_token_us, done_us, prefill_start_us, status,
                                          digest, decisions, evaluations)])
    _check(ctx, lib().asc_simulate_batch(ctx, C.byref(tr), C.byref(oc)), "asc_simulate_batch")


def asc_goodput(ctx, trace_off, arrival_us, output_len, ttft_slo_us, tbt_slo_us, first_token_us,
                done_us, status, good, total, req_ttft_slo_us=None, R=-1):
    T = len(trace_off) - 1
    tr = asc_traces(T, R, _ptr(trace_off), _ptr(arrival_us), None, _ptr(output_len), _ptr(ttft_slo_us),
                    _ptr(tbt_slo_us), _ptr(req_ttft_slo_us))
    oc = asc_outcomes(_ptr(first_token_us), _ptr(done_us), None, _ptr(status), None, None, None)
    _check(ctx, lib().asc_goodput(ctx, C.byref(tr), C.byref(oc), _ptr(good), _ptr(total)),
           "asc_goodput")


def asc_summarize(ctx, trace_off, arrival_us, output_len, ttft_slo_us, tbt_slo_us, first_token_us,
                  done_us, prefill_start_us, status, res, req_ttft_slo_us=None, n_lp=None, R=-1):
    """res: dict SUMMARY_KEY -> int64 [T] array (missing keys are not written)."""
    T = len(trace_off) - 1
    tr = asc_traces(T, R, _ptr(trace_off), _ptr(arrival_us), None, _ptr(output_len), _ptr(ttft_slo_us),
                    _ptr(tbt_slo_us), _ptr(req_ttft_slo_us), _ptr(n_lp))
    oc = asc_outcomes(_ptr(first_token_us), _ptr(done_us), _ptr(prefill_start_us), _ptr(status),
                      None, None, None)
    sm = asc_summary(*[_ptr(res.get(k)) for k in SUMMARY_KEYS])
    _check(ctx, lib().asc_summarize(ctx, C.byref(tr), C.byref(oc), C.byref(sm)), "asc_summarize")


def asc_fit_perf(ctx, rec_off, F, M, y, lam, coef, mean_err=None, max_err=None, N=-1):
    fi = asc_fit_in(len(rec_off) - 1, N, _ptr(rec_off), _ptr(F), _ptr(M), _ptr(y))
    _check(ctx, lib().asc_fit_perf(ctx, C.byref(fi), C.c_double(lam), _ptr(coef), _ptr(mean_err),
                                   _ptr(max_err)), "asc_fit_perf")


def asc_latency(ctx, F, M, lat_us, t_s=None, n=None):
    n = len(F) if n is None else n
    _check(ctx, lib().asc_latency(ctx, C.c_int64(n), _ptr(F), _ptr(M), _ptr(lat_us), _ptr(t_s)), "asc_latency")


# ------------------------------------------------------------------ convenience (allocation) --
class Context:
    """Owns a ctx; allocates outputs as torch CUDA tensors (device path) or numpy (host path)."""

    def __init__(self, cfg, device=0, stream=None):
        self.cfg = cfg
        self.device = device
        self.h = asc_create(cfg, device, stream)

    def close(self):
        if self.h:
            asc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def last_launches(self):
        return asc_last_kernel_launches(self.h)

    def last_kernel_ms(self):
        return asc_last_kernel_ms(self.h)

    def last_kernel2_ms(self):
        return asc_last_kernel2_ms(self.h)

    def arm_snapshots(self, trace, instance, every, max_snaps, entry_cap, out_cap):
        """asc_arm_snapshots with freshly allocated device buffers (returned; read them after the
        next simulate_batch)."""
        import torch
        dev = torch.device("cuda", self.device)
        b = dict(hdr=torch.full((max(max_snaps, 1) * 16,), -1, dtype=torch.int64, device=dev),
                 counts=torch.zeros(3, dtype=torch.int64, device=dev),
                 ids=torch.empty(max(entry_cap, 1), dtype=torch.int32, device=dev),
                 deadline_us=torch.empty(max(entry_cap, 1), dtype=torch.int64, device=dev),
                 eff_prompt=torch.empty(max(entry_cap, 1), dtype=torch.int32, device=dev),
                 flags=torch.empty(max(entry_cap, 1), dtype=torch.uint8, device=dev),
                 out_ids=torch.empty(max(out_cap, 1), dtype=torch.int32, device=dev))
        sn = asc_snapshots(trace, instance, every, max_snaps, entry_cap, out_cap,
                           *[_ptr(b[k]) for k in ("hdr", "counts", "ids", "deadline_us", "eff_prompt",
                                                  "flags", "out_ids")])
        _check(self.h, lib().asc_arm_snapshots(self.h, C.byref(sn)), "asc_arm_snapshots")
        return b

    def schedule_step(self, ins, want_prefill=True, out=None):
        """ins: dict of arrays (all torch CUDA or all numpy).  Returns dict of outputs; `out` (a
        previous call's result for the same shape) is reused instead of allocating."""
        dev = not isinstance(ins["seg_off"], np.ndarray)
        S = len(ins["seg_off"]) - 1
        Q = int(ins["Q"]) if "Q" in ins else int(ins["seg_off"][-1])
        if out is None:
            out = _alloc(dev, self.device, dict(admit_idx=(Q, "i4"), admit_cnt=(S, "i4"),
                                                offload_idx=(Q, "i4"), offload_cnt=(S, "i4"),
                                                drop_idx=(Q, "i4"), drop_cnt=(S, "i4"),
                                                batch_lat_us=(S, "i8"),
                                                prefill_us=(Q if want_prefill else 0, "i4")))
            if not want_prefill:
                out["prefill_us"] = None
        asc_schedule_step(self.h, ins["seg_off"], ins["now_us"], ins["deadline_us"],
                          ins["eff_prompt"], ins["flags"], ins["dec_count"], ins["dec_ctx_sum"],
                          ins["tbt_slo_us"], ins["budget_tokens"], ins["budget_blocks"],
                          ins["budget_reqs"], out["admit_idx"], out["admit_cnt"],
                          out["offload_idx"], out["offload_cnt"], out["drop_idx"],
                          out["drop_cnt"], out["batch_lat_us"], out["prefill_us"], Q=Q)
        return out

    def simulate_batch(self, tr, req_ttft_slo_us=None, out=None, n_lp=None, n_hp=None,
                       req_key_offset_us=None):
        """tr: dict trace_off, arrival_us, prompt_len, output_len, ttft_slo_us, tbt_slo_us;
        n_lp / n_hp: optional per-trace subgroup topology (int32 [T], same kind as tr)."""
        dev = not isinstance(tr["trace_off"], np.ndarray)
        T = len(tr["trace_off"]) - 1
        R = int(tr["R"]) if "R" in tr else int(tr["trace_off"][-1])
        if out is None:
            out = _alloc(dev, self.device, dict(first_token_us=(R, "i8"), done_us=(R, "i8"),
                                                prefill_start_us=(R, "i8"), status=(R, "u4"),
                                                digest=(T, "u8"), decisions=(T, "i8"),
                                                evaluations=(T, "i8")))
        asc_simulate_batch(self.h, tr["trace_off"], tr["arrival_us"], tr["prompt_len"],
                           tr["output_len"], tr["ttft_slo_us"], tr["tbt_slo_us"],
                           out["first_token_us"], out["done_us"], out["prefill_start_us"],
                           out["status"], out["digest"], out["decisions"], out["evaluations"],
                           req_ttft_slo_us, R=R, n_lp=n_lp, n_hp=n_hp,
                           req_key_offset_us=req_key_offset_us)
        return out

    def goodput(self, tr, out, req_ttft_slo_us=None, res=None):
        dev = not isinstance(tr["trace_off"], np.ndarray)
        T = len(tr["trace_off"]) - 1
        if res is None:
            res = _alloc(dev, self.device, dict(good=(T, "u8"), total=(T, "u8")))
        asc_goodput(self.h, tr["trace_off"], tr["arrival_us"], tr["output_len"], tr["ttft_slo_us"],
                    tr["tbt_slo_us"], out["first_token_us"], out["done_us"], out["status"],
                    res["good"], res["total"], req_ttft_slo_us, R=int(tr["R"]) if "R" in tr else -1)
        return res["good"], res["total"]


    def summarize(self, tr, out, req_ttft_slo_us=None, n_lp=None, res=None):
        """Per-trace outcome summary (asc_summarize) -> dict SUMMARY_KEY -> int64 [T]."""
        dev = not isinstance(tr["trace_off"], np.ndarray)
        T = len(tr["trace_off"]) - 1
        if res is None:
            res = _alloc(dev, self.device, {k: (T, "i8") for k in SUMMARY_KEYS})
        asc_summarize(self.h, tr["trace_off"], tr["arrival_us"], tr["output_len"], tr["ttft_slo_us"],
                      tr["tbt_slo_us"], out["first_token_us"], out["done_us"], out["prefill_start_us"],
                      out["status"], res, req_ttft_slo_us, n_lp, R=int(tr["R"]) if "R" in tr else -1)
        return {k: v[:T] for k, v in res.items()}

    def fit_perf(self, rec, lam=1e-8, errors=True):
        """rec: dict(off, F, M, y) numpy (host path) or torch CUDA tensors (device path)
        -> (coef [G, 5], mean_err [G] or None, max_err [G] or None), same kind as the input."""
        dev = not isinstance(rec["off"], np.ndarray)
        G = len(rec["off"]) - 1
        if dev:
            import torch
            mk = lambda n: torch.empty(max(n, 1), dtype=torch.float64, device=f"cuda:{self.device}")
        else:
            mk = lambda n: np.zeros(max(n, 1), np.float64)
        coef = mk(5 * G)
        me, mx = (mk(G), mk(G)) if errors else (None, None)
        N = int(rec["N"]) if "N" in rec else -1
        asc_fit_perf(self.h, rec["off"], rec["F"], rec["M"], rec["y"], lam, coef, me, mx, N=N)
        coef = coef[:5 * G].reshape(G, 5)
        return coef, (me[:G] if errors else None), (mx[:G] if errors else None)


def _latency_method(self, F, M, want_t=True):
    """Eq. 4-5 latency of n batches from their (F, M) (uint64 numpy, or int64/uint64 torch CUDA
    tensors) -> (lat_us int64 [n], t_s float64 [n] or None), same kind as the input."""
    dev = not isinstance(F, np.ndarray)
    n = len(F)
    if dev:
        import torch
        lat = torch.empty(max(n, 1), dtype=torch.int64, device=f"cuda:{self.device}")
        ts = torch.empty(max(n, 1), dtype=torch.float64, device=f"cuda:{self.device}") if want_t else None
    else:
        lat = np.zeros(max(n, 1), np.int64)
        ts = np.zeros(max(n, 1), np.float64) if want_t else None
    asc_latency(self.h, F, M, lat, ts, n=n)
    return lat[:n], (ts[:n] if want_t else None)


Context.latency = _latency_method


def _alloc(dev, device, spec):
    if not dev:
        return {k: np.zeros(max(n, 1), dtype=dt) for k, (n, dt) in spec.items()}
    import torch
    tmap = {"i4": torch.int32, "i8": torch.int64, "u4": torch.int32, "u8": torch.int64}
    return {k: torch.empty(max(n, 1), dtype=tmap[dt], device=f"cuda:{device}")
            for k, (n, dt) in spec.items()}


def batch_arrays(batch, device=None):
    """gen.traces.TraceBatch -> dict of numpy (host) or torch CUDA tensors (device)."""
    d = dict(trace_off=batch.trace_off, arrival_us=batch.arrival_us, prompt_len=batch.prompt_len,
             output_len=batch.output_len, ttft_slo_us=batch.ttft_slo_us, tbt_slo_us=batch.tbt_slo_us)
    # zero-length arrays would marshal as NULL: pad to one (never read) element
    d = {k: np.ascontiguousarray(v if len(v) else np.zeros(1, v.dtype)) for k, v in d.items()}
    R = int(batch.trace_off[-1])
    if device is None:
        d["R"] = R
        return d
    import torch
    d = {k: torch.from_numpy(v).to(device) for k, v in d.items()}
    d["R"] = R  # host-known total so the library needs no device->host read
    return d
