"""ctypes wrapper of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module.  It loads oracle/liboracle.so (built by `make -C oracle`
or __graft_entry__.build()) and marshals numpy arrays; all arithmetic is in oracle.cpp.
"""
import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class OrArch(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("h", "n", "s", "n_kv", "m", "L", "b", "d", "tp")]


class OrPerf(C.Structure):
    _fields_ = [("c", C.c_double * 5), ("F_H", C.c_double), ("M_H", C.c_double)]


class OrSched(C.Structure):
    _fields_ = ([(k, C.c_int32) for k in ("n_lp", "n_hp", "bs", "kv_lp", "kv_hp", "lp_max_batch",
                                          "lp_tok", "hp_tok", "policy", "offload", "tickets",
                                          "elastic", "drop", "hist_default")]
                + [("margin_us", C.c_int64), ("delay_us", C.c_int64), ("scheduler", C.c_int32),
                   ("chunk_tokens", C.c_int32), ("offload_rule", C.c_int32),
                   ("key_w", C.c_int32 * 3)])


def build():
    subprocess.check_call(["make", "-s", "-C", _HERE])


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        src = os.path.join(_HERE, "oracle.cpp")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            build()
        _LIB = C.CDLL(path)
        _LIB.or_latency_s.restype = C.c_double
        _LIB.or_latency_us.restype = C.c_int64
        _LIB.or_batch_us.restype = C.c_int64
        _LIB.or_algorithm1.restype = C.c_int32
        _LIB.or_last_error.restype = C.c_char_p
    return _LIB


def arch_s(a):
    return OrArch(a["h"], a["n"], a["s"], a["n_kv"], a["m"], a["L"], a["b"], a["dtype_bytes"], a["tp"])


def perf_s(p):
    return OrPerf((C.c_double * 5)(*p["c"]), p["F_H"], p["M_H"])


def sched_s(cfg):
    t, f = cfg["topo"], cfg["flags"]
    return OrSched(t["n_lp"], t["n_hp"], t["block_tokens"], t["kv_blocks_lp"], t["kv_blocks_hp"],
                   t["lp_max_batch"], t["lp_token_budget"], t["hp_token_budget"], f["policy"],
                   f["offload"], f["tickets"], f["elastic"], f["drop"], f["hist_default_tokens"],
                   f["offload_margin_us"], f["offload_delay_us"], f.get("scheduler", 0),
                   f.get("chunk_tokens", 512), f.get("offload_rule", 0),
                   (C.c_int32 * 3)(*f.get("key_weights", (1, -1, 0))))


def _p(a, dt):
    a = np.ascontiguousarray(a, dtype=dt)
    return a, a.ctypes.data_as(C.c_void_p)


def _err():
    return lib().or_last_error().decode()


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def cost(arch, p, lhat=()):
    pa, pp = _p(p, np.int64)
    la, lp = _p(lhat, np.int64)
    F, M = C.c_uint64(), C.c_uint64()
    a = arch_s(arch)
    rc = lib().or_cost(C.byref(a), len(pa), pp, len(la), lp, C.byref(F), C.byref(M))
    return F.value, M.value, rc


def cost_chunked(arch, l, c, lhat=()):
    la_, lp_ = _p(l, np.int64)
    ca, cp = _p(c, np.int64)
    da, dp = _p(lhat, np.int64)
    assert len(la_) == len(ca)
    F, M = C.c_uint64(), C.c_uint64()
    a = arch_s(arch)
    rc = lib().or_cost_chunked(C.byref(a), len(ca), lp_, cp, len(da), dp, C.byref(F), C.byref(M))
    return F.value, M.value, rc


def fit_perf(perf, off, F, M, y, lam=1e-8, errors=True):
    """-> (coef [G, 5], mean_err [G], max_err [G]) of the ridge fit (or_fit_perf)."""
    offa, offp = _p(off, np.int64)
    Fa, Fp = _p(F, np.uint64)
    Ma, Mp = _p(M, np.uint64)
    ya, yp = _p(y, np.float64)
    G = len(offa) - 1
    coef = np.zeros((max(G, 1), 5))
    me, mx = np.zeros(max(G, 1)), np.zeros(max(G, 1))
    ps = perf_s(perf)
    rc = lib().or_fit_perf(C.byref(ps), G, offp, Fp, Mp, yp, C.c_double(lam),
                           coef.ctypes.data_as(C.c_void_p),
                           me.ctypes.data_as(C.c_void_p) if errors else None,
                           mx.ctypes.data_as(C.c_void_p) if errors else None)
    if rc:
        raise OracleError(rc, _err())
    return coef[:G], me[:G], mx[:G]


def latency_s(perf, F, M):
    ps = perf_s(perf)
    return lib().or_latency_s(C.byref(ps), C.c_uint64(F), C.c_uint64(M))


def latency_us(perf, F, M):
    ps = perf_s(perf)
    return lib().or_latency_us(C.byref(ps), C.c_uint64(F), C.c_uint64(M))


def latency_n(perf, F, M):
    """(lat_us int64 [n], t seconds float64 [n]) of n (F, M) pairs via or_latency_n."""
    F = np.ascontiguousarray(F, dtype=np.uint64)
    M = np.ascontiguousarray(M, dtype=np.uint64)
    n = len(F)
    lat = np.zeros(n, np.int64)
    t = np.zeros(n, np.float64)
    ps = perf_s(perf)
    lib().or_latency_n(C.byref(ps), C.c_int64(n), F.ctypes.data_as(C.c_void_p), M.ctypes.data_as(C.c_void_p),
                       lat.ctypes.data_as(C.c_void_p), t.ctypes.data_as(C.c_void_p))
    return lat, t


def batch_us(arch, perf, p, lhat=()):
    pa, pp = _p(p, np.int64)
    la, lp = _p(lhat, np.int64)
    a, ps = arch_s(arch), perf_s(perf)
    return lib().or_batch_us(C.byref(a), C.byref(ps), len(pa), pp, len(la), lp)


INF = (1 << 63) - 1


def algorithm1(val, ids, c, mem, tok, Cb, Mb, Nb, Rb):
    n = len(val)
    arrs = [_p(x, np.int64) for x in (val, ids, c, mem, tok)]
    sel = np.zeros(max(n, 1), np.int32)
    k = lib().or_algorithm1(n, *[x[1] for x in arrs], C.c_int64(Cb), C.c_int64(Mb),
                            C.c_int64(Nb), C.c_int64(Rb), sel.ctypes.data_as(C.c_void_p))
    return [int(x) for x in sel[:k]]


def schedule_step(cfg, seg_off, now_us, deadline_us, eff_prompt, flags, dec_count, dec_ctx_sum,
                  tbt_slo_us, budget_tokens, budget_blocks, budget_reqs):
    seg_off = np.ascontiguousarray(seg_off, np.int64)
    S = len(seg_off) - 1
    Q = int(seg_off[-1])
    ins = [_p(x, dt) for x, dt in ((seg_off, np.int64), (now_us, np.int64),
                                   (deadline_us, np.int64), (eff_prompt, np.int32),
                                   (flags, np.uint8), (dec_count, np.int32),
                                   (dec_ctx_sum, np.int64), (tbt_slo_us, np.int64),
                                   (budget_tokens, np.int32), (budget_blocks, np.int32),
                                   (budget_reqs, np.int32))]
    out = dict(admit_idx=np.zeros(max(Q, 1), np.int32), admit_cnt=np.zeros(S, np.int32),
               offload_idx=np.zeros(max(Q, 1), np.int32), offload_cnt=np.zeros(S, np.int32),
               drop_idx=np.zeros(max(Q, 1), np.int32), drop_cnt=np.zeros(S, np.int32),
               batch_lat_us=np.zeros(S, np.int64), prefill_us=np.zeros(max(Q, 1), np.int32))
    a, ps, sc = arch_s(cfg["arch"]), perf_s(cfg["perf"]), sched_s(cfg)
    rc = lib().or_schedule_step(C.byref(a), C.byref(ps), C.byref(sc), S, *[x[1] for x in ins],
                                *[out[k].ctypes.data_as(C.c_void_p) for k in
                                  ("admit_idx", "admit_cnt", "offload_idx", "offload_cnt",
                                   "drop_idx", "drop_cnt", "batch_lat_us", "prefill_us")])
    if rc:
        raise OracleError(rc, _err())
    out["prefill_us"] = out["prefill_us"][:Q]
    return out


def simulate_batch(cfg, batch, req_ttft_slo_us=None, nthreads=0, check_invariants=False,
                   n_lp=None, n_hp=None, req_key_offset_us=None):
    """batch: gen.traces.TraceBatch; n_lp / n_hp: optional per-trace subgroup topology (row f3).
    Returns dict of per-request and per-trace outputs."""
    T, R = batch.T, batch.R
    ins = [_p(x, dt) for x, dt in ((batch.trace_off, np.int64), (batch.arrival_us, np.int64),
                                   (batch.prompt_len, np.int32), (batch.output_len, np.int32),
                                   (batch.ttft_slo_us, np.int64), (batch.tbt_slo_us, np.int64))]
    rt = None
    if req_ttft_slo_us is not None:
        rt = _p(req_ttft_slo_us, np.int64)
    out = dict(first_token_us=np.zeros(max(R, 1), np.int64), done_us=np.zeros(max(R, 1), np.int64),
               prefill_start_us=np.zeros(max(R, 1), np.int64),
               status=np.zeros(max(R, 1), np.uint32), digest=np.zeros(max(T, 1), np.uint64),
               decisions=np.zeros(max(T, 1), np.int64), evaluations=np.zeros(max(T, 1), np.int64))
    a, ps, sc = arch_s(cfg["arch"]), perf_s(cfg["perf"]), sched_s(cfg)
    nl = _p(n_lp, np.int32) if n_lp is not None else None
    nh = _p(n_hp, np.int32) if n_hp is not None else None
    ko = _p(req_key_offset_us, np.int64) if req_key_offset_us is not None else None
    rc = lib().or_simulate_batch(C.byref(a), C.byref(ps), C.byref(sc), T, *[x[1] for x in ins],
                                 rt[1] if rt else None, nl[1] if nl else None, nh[1] if nh else None,
                                 ko[1] if ko else None,
                                 *[out[k].ctypes.data_as(C.c_void_p) for k in
                                   ("first_token_us", "done_us", "prefill_start_us", "status",
                                    "digest", "decisions", "evaluations")],
                                 int(nthreads), int(bool(check_invariants)))
    if rc:
        raise OracleError(rc, _err())
    for k in ("first_token_us", "done_us", "prefill_start_us", "status"):
        out[k] = out[k][:R]
    for k in ("digest", "decisions", "evaluations"):
        out[k] = out[k][:T]
    return out


def goodput(batch, out, req_ttft_slo_us=None):
    T = batch.T
    good = np.zeros(max(T, 1), np.uint64)
    total = np.zeros(max(T, 1), np.uint64)
    ins = [_p(x, dt) for x, dt in ((batch.trace_off, np.int64), (batch.arrival_us, np.int64),
                                   (batch.output_len, np.int32), (batch.ttft_slo_us, np.int64),
                                   (batch.tbt_slo_us, np.int64))]
    rt = _p(req_ttft_slo_us, np.int64) if req_ttft_slo_us is not None else None
    outs = [_p(out[k], dt) for k, dt in (("first_token_us", np.int64), ("done_us", np.int64),
                                        ("status", np.uint32))]
    rc = lib().or_goodput(T, *[x[1] for x in ins], rt[1] if rt else None, *[x[1] for x in outs],
                          good.ctypes.data_as(C.c_void_p), total.ctypes.data_as(C.c_void_p))
    if rc:
        raise OracleError(rc, _err())
    return good[:T], total[:T]


SUMMARY_KEYS = ("completed", "dropped", "violating", "tokens", "ttft_p50_us", "ttft_p90_us",
                "ttft_p99_us", "tbt_sum_us", "tbt_tokens", "delay_sum_lp_us", "delay_cnt_lp",
                "delay_sum_hp_us", "delay_cnt_hp", "last_done_us")


def summarize(cfg, batch, out, req_ttft_slo_us=None, n_lp=None):
    """Per-trace outcome summary (or_summarize; row a8): dict of int64 [T] arrays, SUMMARY_KEYS."""
    T = batch.T
    ins = [_p(x, dt) for x, dt in ((batch.trace_off, np.int64), (batch.arrival_us, np.int64),
                                   (batch.output_len, np.int32), (batch.ttft_slo_us, np.int64),
                                   (batch.tbt_slo_us, np.int64))]
    rt = _p(req_ttft_slo_us, np.int64) if req_ttft_slo_us is not None else None
    nl = _p(n_lp, np.int32) if n_lp is not None else None
    outs = [_p(out[k], dt) for k, dt in (("first_token_us", np.int64), ("done_us", np.int64),
                                        ("prefill_start_us", np.int64), ("status", np.uint32))]
    res = {k: np.zeros(max(T, 1), np.int64) for k in SUMMARY_KEYS}
    rc = lib().or_summarize(T, *[x[1] for x in ins], rt[1] if rt else None, nl[1] if nl else None,
                            int(cfg["topo"]["n_lp"]), *[x[1] for x in outs],
                            *[res[k].ctypes.data_as(C.c_void_p) for k in SUMMARY_KEYS])
    if rc:
        raise OracleError(rc, _err())
    return {k: v[:T] for k, v in res.items()}


# status word layout
def state(st):
    return np.asarray(st) & 3


def instance(st):
    return (np.asarray(st) >> 4) & 255


def preemptions(st):
    return (np.asarray(st) >> 12) & 0xFFFF
