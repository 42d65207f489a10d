"""Seeded synthetic request traces (INPUT GENERATOR ONLY).

This module is the one piece shared by the oracle tests and the CUDA path: it
draws arrivals and prompt/output lengths and holds none of the method's
arithmetic (no cost model, no priorities, no scheduling).  Everything is
integer: a counter-based splitmix64 stream indexes 65,536-entry quantile
tables (gen/tables.npz, written by gen/make_tables.py).

Recipe:
  seed_trace = mix(base_seed ^ trace_idx)
  u(i, σ)    = mix(seed_trace + (3 i + σ) * 0x9E3779B97F4A7C15),  σ ∈ {0 gap, 1 prompt, 2 output}
  prompt_i   = prompt_table[u(i,1) >> 48], output_i = output_table[u(i,2) >> 48]
  gap_i      = ((exp_q32[u(i,0) >> 48] * 8_000_000) // qps_j) >> 32     (QPS = qps_j / 8; Poisson)
  arrival_i  = arrival_{i-1} + gap_i,  arrival_{-1} = 0                    (integer microseconds)
"""
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_TABLES = None

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def tables():
    global _TABLES
    if _TABLES is None:
        with np.load(os.path.join(_HERE, "tables.npz")) as z:
            _TABLES = {k: z[k] for k in z.files}
    return _TABLES


def mix_np(x):
    """splitmix64 finalizer on a uint64 ndarray (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def mix_int(x):
    """splitmix64 finalizer on a Python int (reference for tests of the generator)."""
    x &= M64
    z = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


SHAPES = {
    "sharegpt": ("sharegpt_prompt", "sharegpt_output"),
    "longbench": ("longbench_prompt", "longbench_output"),
}


def gen_trace(base_seed, trace_idx, shape, qps_j, n):
    """One trace of n requests: (arrival_us int64[n], prompt int32[n], output int32[n])."""
    if n == 0:
        return (np.zeros(0, np.int64), np.zeros(0, np.int32), np.zeros(0, np.int32))
    t = tables()
    pt, ot = SHAPES[shape]
    seed = mix_int((base_seed ^ trace_idx) & M64)
    i = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        base = np.uint64(seed) + np.uint64(3) * i * np.uint64(GOLDEN)
        u_gap = mix_np(base)
        u_pr = mix_np(base + np.uint64(GOLDEN))
        u_out = mix_np(base + np.uint64(2) * np.uint64(GOLDEN))
    s48 = np.uint64(48)
    e = t["exp_q32"][(u_gap >> s48).astype(np.int64)]
    gap = ((e * np.uint64(8_000_000)) // np.uint64(qps_j)) >> np.uint64(32)
    arrival = np.cumsum(gap.astype(np.int64))
    prompt = t[pt][(u_pr >> s48).astype(np.int64)].astype(np.int32)
    output = t[ot][(u_out >> s48).astype(np.int64)].astype(np.int32)
    return arrival.astype(np.int64), prompt, output


@dataclass
class TraceBatch:
    """CSR batch of independent traces (host numpy arrays)."""
    trace_off: np.ndarray      # int64 [T+1]
    arrival_us: np.ndarray     # int64 [R]
    prompt_len: np.ndarray     # int32 [R]
    output_len: np.ndarray     # int32 [R]
    ttft_slo_us: np.ndarray    # int64 [T]
    tbt_slo_us: np.ndarray     # int64 [T]
    qps_j: np.ndarray          # int32 [T]   (QPS = qps_j / 8)
    labels: list               # per-trace description

    @property
    def T(self):
        return len(self.trace_off) - 1

    @property
    def R(self):
        return int(self.trace_off[-1])

    def trace(self, t):
        a, b = int(self.trace_off[t]), int(self.trace_off[t + 1])
        return (self.arrival_us[a:b], self.prompt_len[a:b], self.output_len[a:b],
                int(self.ttft_slo_us[t]), int(self.tbt_slo_us[t]))

    def subset(self, idx):
        parts = [self.trace(int(t)) for t in idx]
        return make_batch([(p[0], p[1], p[2]) for p in parts],
                          [p[3] for p in parts], [p[4] for p in parts],
                          [int(self.qps_j[int(t)]) for t in idx],
                          [self.labels[int(t)] for t in idx])


def make_batch(traces, ttft, tbt, qps_j=None, labels=None):
    T = len(traces)
    lens = np.array([len(tr[0]) for tr in traces], dtype=np.int64)
    off = np.zeros(T + 1, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    cat = lambda k, dt: (np.concatenate([np.asarray(tr[k], dtype=dt) for tr in traces])
                         if T else np.zeros(0, dt))
    return TraceBatch(off, cat(0, np.int64), cat(1, np.int32), cat(2, np.int32),
                      np.asarray(ttft, dtype=np.int64), np.asarray(tbt, dtype=np.int64),
                      np.asarray(qps_j if qps_j is not None else [0] * T, dtype=np.int32),
                      list(labels) if labels is not None else [""] * T)


def grid_batch(points, n, shape, base_ttft, base_tbt, base_seed=1):
    """points: list of (trace_idx, qps_j, scale_num, scale_den).  SLO scale applied exactly."""
    trs, tt, tb, qj, lab = [], [], [], [], []
    for (tidx, j, num, den) in points:
        trs.append(gen_trace(base_seed, tidx, shape, j, n))
        assert (base_ttft * num) % den == 0 and (base_tbt * num) % den == 0
        tt.append(base_ttft * num // den)
        tb.append(base_tbt * num // den)
        qj.append(j)
        lab.append(f"t{tidx}:qps{j}/8:slo{num}/{den}")
    return make_batch(trs, tt, tb, qj, lab)
