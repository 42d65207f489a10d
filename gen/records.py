"""Synthetic batch-latency records for the Eq. 4-5 calibration (row f2) — INPUT DATA ONLY.

A record is what the paper's runtime logs per executed batch: the batch's exact flop
count F and byte count M (integers, as the cost model would give) and an "observed" latency in
seconds.  Both sides read the same arrays.  The observed latency is a stand-in for a measurement:
bytes over a nominal 1.6 TB/s plus 0.2 ms, with a counter-based multiplicative noise term — no
Eq. 4-5 arithmetic (features, max, coefficients) happens here.

Per record i of group g (counter-based, splitmix64 as in traces.py):
  u_k = mix(seed_g + (4i + k) * GOLD), k = 0..3, seed_g = mix(base_seed ^ (g + 0x5EED))
  M = 10^9 * 2^(u_0 / 2^64 * 7.5)      (1 GB .. ~181 GB, log-uniform)
  F = 10^10 * 2^(u_1 / 2^64 * 16)      (1e10 .. 6.5e14 flops, log-uniform)
  y = (M / 1.6e12 + 2e-4) * (1 + noise * (u_2 / 2^64 - 0.5) * 2)
"""
import numpy as np

from .traces import mix_np

GOLD = np.uint64(0x9E3779B97F4A7C15)


def group_records(base_seed, g, n, noise=0.05):
    i = np.arange(n, dtype=np.uint64)
    seed = mix_np(np.uint64(base_seed) ^ np.uint64(g + 0x5EED))
    with np.errstate(over="ignore"):
        u = [mix_np(seed + (np.uint64(4) * i + np.uint64(k)) * GOLD) for k in range(3)]
    f = [x.astype(np.float64) / 2.0 ** 64 for x in u]
    M = np.floor(1e9 * np.exp2(f[0] * 7.5)).astype(np.uint64)
    F = np.floor(1e10 * np.exp2(f[1] * 16.0)).astype(np.uint64)
    y = (M.astype(np.float64) / 1.6e12 + 2e-4) * (1.0 + noise * (f[2] - 0.5) * 2.0)
    return F, M, y


def make_records(base_seed, sizes, noise=0.05):
    """sizes: records per group -> dict(off, F, M, y) as contiguous numpy arrays (CSR by group)."""
    off = np.zeros(len(sizes) + 1, np.int64)
    off[1:] = np.cumsum(sizes)
    parts = [group_records(base_seed, g, int(n), noise) for g, n in enumerate(sizes)]
    cat = lambda k, dt: (np.concatenate([p[k] for p in parts]).astype(dt) if parts else np.zeros(0, dt))
    return dict(off=off, F=cat(0, np.uint64), M=cat(1, np.uint64), y=cat(2, np.float64))
