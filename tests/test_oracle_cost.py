"""Pins for the oracle's performance model (Eq. 1-7, App. A).

Each test checks the oracle against something other than itself: the SPEC's hand
evaluations, the closed form of the TINY-LINEAR preset, the printed Eq. 6/7 (a different
passage from the Table 3/4 row sums the oracle is written from), reductions and scaling.
"""
import math

import numpy as np
import pytest

from gen import presets as P

TOY = dict(h=4, n=2, s=2, n_kv=2, m=8, L=1, b=2, dtype_bytes=1, tp=1)


def test_spec_prefill_worked_value(oracle):
    # S:67 [DERIVED]: (h=4,n=2,s=2,m=8,b=2,L=1,d=1; p=[2]) -> F = 256 + 32 = 288; M = 224 + 40 = 264
    assert oracle.cost(TOY, [2])[:2] == (288, 264)


def test_spec_decode_worked_value(oracle):
    # S:77 [DERIVED]: lhat=[3] -> F = 128 + 24 = 152; M = 176 + 32 = 208
    assert oracle.cost(TOY, [], [3])[:2] == (152, 208)


def eq6_eq7(a, p, lhat):
    """PAPER.md Eq. 6 and Eq. 7 as printed, merged per Eq. 8/9's
    hybrid form (weights once, G8), with the per-request sums and head factor n of Eq. 3
    (G4) and ceil(p/b) (G9).  Written independently of the oracle's Table-3/4 row sums."""
    h, n, s, m, b, L, d = a["h"], a["n"], a["s"], a["m"], a["b"], a["L"], a["dtype_bytes"]
    t = sum(p)
    Bd = len(lhat)
    nonempty = 1 if (p or lhat) else 0
    M = nonempty * (4 * h * h + 2 * h * m) + 8 * t * h + 2 * t * m \
        + n * sum(2 * s * q + 3 * s * q * (-(-q // b)) for q in p) \
        + 8 * Bd * h + 2 * Bd * m + n * sum(2 * l * s + 2 * s for l in lhat)
    F = 4 * t * h * h + 2 * t * h * m + n * sum(2 * q * q * s for q in p) \
        + 4 * Bd * h * h + 2 * Bd * h * m + n * sum(2 * l * s for l in lhat)
    return F * L, M * L * d


@pytest.mark.parametrize("seed", range(5))
def test_table_rows_equal_printed_equations(oracle, seed):
    rng = np.random.default_rng(seed)
    for _ in range(200):
        n = int(rng.integers(1, 9))
        s = int(rng.integers(1, 9))
        a = dict(h=n * s, n=n, s=s, n_kv=1, m=int(rng.integers(1, 50)), L=int(rng.integers(1, 5)),
                 b=int(rng.integers(1, 40)), dtype_bytes=int(rng.integers(1, 3)), tp=1)
        p = [int(x) for x in rng.integers(1, 300, size=int(rng.integers(0, 5)))]
        lh = [int(x) for x in rng.integers(1, 3000, size=int(rng.integers(0, 5)))]
        F, M, rc = oracle.cost(a, p, lh)
        assert rc == 0
        assert (F, M) == eq6_eq7(a, p, lh)


def test_tiny_linear_closed_form(oracle):
    # TINY-LINEAR: lat (s) = M = 6 + 15 sum(p) + 12 B_d + 2 sum(lhat) exactly (SURVEY c.11)
    rng = np.random.default_rng(7)
    for _ in range(300):
        p = [int(x) for x in rng.integers(1, 1000, size=int(rng.integers(0, 6)))]
        lh = [int(x) for x in rng.integers(1, 5000, size=int(rng.integers(0, 6)))]
        if not p and not lh:
            continue
        expect = 6 + 15 * sum(p) + 12 * len(lh) + 2 * sum(lh)
        assert oracle.batch_us(P.TINY, P.PERF_TINY, p, lh) == expect * 1_000_000


def test_reductions_and_scaling(oracle):
    a = dict(P.MISTRAL7B)
    p, lh = [513, 77], [1000, 2048, 5]
    Fh, Mh, _ = oracle.cost(a, p, lh)
    Fp, Mp, _ = oracle.cost(a, p, [])
    Fd, Md, _ = oracle.cost(a, [], lh)
    wF, wM = 0, (4 * a["h"] ** 2 + 2 * a["h"] * a["m"]) * a["L"] * a["dtype_bytes"]
    # hybrid = prefill + decode with the weight read counted once (G8)
    assert Fh == Fp + Fd - wF and Mh == Mp + Md - wM
    a2 = dict(a, L=2 * a["L"])
    assert oracle.cost(a2, p, lh)[:2] == (2 * Fh, 2 * Mh)
    a3 = dict(a, dtype_bytes=2 * a["dtype_bytes"])
    assert oracle.cost(a3, p, lh)[:2] == (Fh, 2 * Mh)
    # monotone: adding a request strictly increases F and M
    F2, M2, _ = oracle.cost(a, p + [1], lh)
    assert F2 > Fh and M2 > Mh
    F3, M3, _ = oracle.cost(a, p, lh + [1])
    assert F3 > Fh and M3 > Mh
    # decode cost depends on the contexts only through their sum (Eq. 2 is linear)
    assert oracle.cost(a, [], [1000, 2048, 5])[:2] == oracle.cost(a, [], [3051, 1, 1])[:2]


def test_tp_division(oracle):
    # App. A.1 note: h, n, m divided by the TP degree
    a = dict(P.MISTRAL7B, tp=2)
    b = dict(P.MISTRAL7B, h=2048, n=16, m=7168, n_kv=4, tp=1)
    cfg_a = P.config(arch=a)
    cfg_b = P.config(arch=b)
    ins = dict(seg_off=[0, 1], now_us=[0], deadline_us=[10 ** 7], eff_prompt=[700], flags=[0],
               dec_count=[0], dec_ctx_sum=[0], tbt_slo_us=[0], budget_tokens=[8192],
               budget_blocks=[100], budget_reqs=[4])
    ra = oracle.schedule_step(cfg_a, **ins)
    rb = oracle.schedule_step(cfg_b, **ins)
    assert ra["prefill_us"][0] == rb["prefill_us"][0] == oracle.batch_us(b, P.PERF_ROOFLINE, [700])


def test_latency_spec_examples(oracle):
    # features t_M=2, t_F=3 via M=2 M_H, F=3 F_H
    pf = dict(c=(0, 1, 0, 0, 0), F_H=1e12, M_H=1e12)
    assert oracle.latency_s(pf, 3 * 10 ** 12, 2 * 10 ** 12) == 3.0
    pf = dict(c=(1, 0, 0, 0, 0), F_H=1e15, M_H=1e15)
    assert oracle.latency_s(pf, 3 * 10 ** 12, 2 * 10 ** 12) == pytest.approx(0.005, rel=1e-15)
    pf = dict(c=(0, 0, 0, 0, 0.25), F_H=1.0, M_H=1.0)
    assert oracle.latency_s(pf, 123, 456) == 0.25
    # unit normalisation F = F_H, M = M_H -> features (2,1,1,1,1): sum of coefficients
    pf = dict(c=(1, 10, 100, 1000, 10000), F_H=1e6, M_H=1e6)
    assert oracle.latency_s(pf, 10 ** 6, 10 ** 6) == 2 + 10 + 100 + 1000 + 10000


def test_latency_clamp_and_floor(oracle):
    # negative prediction clamps to 0; G17: event time floors at 1 microsecond
    pf = dict(c=(0, 0, 0, 0, -1.0), F_H=1.0, M_H=1.0)
    assert oracle.latency_s(pf, 5, 5) == 0.0
    assert oracle.latency_us(pf, 5, 5) == 1
    # G18: ceil to the next microsecond
    pf = dict(c=(0, 0, 0, 0, 1.0000001e-6 + 0.0), F_H=1.0, M_H=1.0)
    assert oracle.latency_us(pf, 0, 0) == 2
    pf = dict(c=(0, 0, 1, 0, 0), F_H=1.0, M_H=4e6)
    assert oracle.latency_us(pf, 0, 10) == math.ceil(10 / 4e6 * 1e6)


def test_range_guard(oracle):
    # F or M at or above 2^53 is not exactly representable: flagged
    a = dict(P.MISTRAL7B, L=10 ** 6)
    assert oracle.cost(a, [32768])[2] == 1
    assert oracle.cost(P.MISTRAL7B, [32768])[2] == 0


def test_range_guard_catches_uint64_wrap(oracle):
    # F is checked against 2^53 after uint64 products; with powers of two chosen so
    # that the exact F is 2^73 + 3 * 2^66 (a multiple of 2^64), the wrapped product is exactly 0 --
    # "in range" without a guard.  The fp64 shadow flags it.
    a = dict(h=1 << 16, n=1 << 8, s=1 << 8, n_kv=1 << 8, m=1 << 16, L=1 << 10, b=1, dtype_bytes=2, tp=1)
    p = 1 << 23
    exact_F = a["L"] * (p * (4 * a["h"] ** 2 + 2 * a["h"] * a["m"]) + a["n"] * 2 * a["s"] * p * p)
    assert exact_F % (1 << 64) == 0 and exact_F >= 1 << 53
    F, M, rc = oracle.cost(a, [p])
    assert rc == 1


def test_step_rejects_eff_prompt_at_2_24(oracle):
    # eff_prompt >= 2^24 is out of range for asc_schedule_step (include/asc.h)
    cfg = P.config()
    ins = dict(seg_off=np.array([0, 2], np.int64), now_us=np.array([10 ** 7], np.int64),
               deadline_us=np.array([10 ** 7, 10 ** 7], np.int64),
               eff_prompt=np.array([100, 1 << 24], np.int32), flags=np.zeros(2, np.uint8),
               dec_count=np.zeros(1, np.int32), dec_ctx_sum=np.zeros(1, np.int64),
               tbt_slo_us=np.array([150000], np.int64), budget_tokens=np.array([8192], np.int32),
               budget_blocks=np.array([25000], np.int32), budget_reqs=np.array([128], np.int32))
    with pytest.raises(oracle.OracleError) as e:
        oracle.schedule_step(cfg, **ins)
    assert e.value.code == 6


def test_latency_batch_wrapper(oracle):
    # or_latency_n is a loop over or_latency_us / or_latency_s (the GPU latency test's reference)
    rng = np.random.default_rng(8)
    pf = dict(c=(0.1, 0.9, 0.05, -0.02, 3e-4), F_H=312e12, M_H=2e12)
    F = (2.0 ** rng.uniform(0, 53, 500)).astype(np.uint64)
    M = (2.0 ** rng.uniform(0, 53, 500)).astype(np.uint64)
    lat, t = oracle.latency_n(pf, F, M)
    for i in range(500):
        assert lat[i] == oracle.latency_us(pf, int(F[i]), int(M[i]))
        assert t[i] == oracle.latency_s(pf, int(F[i]), int(M[i]))
