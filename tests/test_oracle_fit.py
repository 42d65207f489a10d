"""Pins for the oracle's Eq. 4-5 calibration (row f2; G49).

Round trip: records synthesised from known coefficients through the Eq. 4-5 predictor are fitted
back to predictions within 1e-6 relative; the regularised normal equations agree with an
independent numpy solve; held-out error under 5% noise is below 10% (Fig. 7); exact
special cases (intercept-only, pure max); S:154's minimum group size.
"""
import numpy as np
import pytest

from gen import presets as P
from gen import records as RC

PERF = P.PERF_ROOFLINE


def _truth(oracle, c, F, M):
    pf = dict(PERF, c=tuple(c))
    return np.array([oracle.latency_s(pf, int(f), int(m)) for f, m in zip(F, M)])


def _pred(oracle, c, F, M):
    return _truth(oracle, c, F, M)


@pytest.mark.parametrize("c", [(0.0, 1.0, 0.0, 0.0, 3e-4), (0.3, 0.5, 0.2, 0.1, 1e-4),
                               (0.0, 0.0, 1.1, 0.9, 0.0), (0.0, 0.0, 0.0, 0.0, 0.25)])
def test_round_trip_noise_free(oracle, c):
    r = RC.make_records(3, [400])
    y = _truth(oracle, c, r["F"], r["M"])
    coef, me, mx = oracle.fit_perf(PERF, r["off"], r["F"], r["M"], y)
    pred = _pred(oracle, coef[0], r["F"], r["M"])
    assert np.max(np.abs(pred - y) / y) < 1e-6
    assert mx[0] < 1e-6 and me[0] <= mx[0]


def test_matches_independent_numpy_solve(oracle):
    r = RC.make_records(4, [500, 37, 2000])
    coef, _, _ = oracle.fit_perf(PERF, r["off"], r["F"], r["M"], r["y"], lam=1e-8, errors=False)
    for g in range(3):
        lo, hi = r["off"][g], r["off"][g + 1]
        tM = r["M"][lo:hi].astype(np.float64) / PERF["M_H"]
        tF = r["F"][lo:hi].astype(np.float64) / PERF["F_H"]
        X = np.stack([tM + tF, np.maximum(tM, tF), tM, tF, np.ones_like(tM)], 1)
        A = X.T @ X + 1e-8 * np.eye(5)
        c = np.linalg.solve(A, X.T @ r["y"][lo:hi])
        # predictions, not coefficients: x1 = x3 + x4 makes the unregularised system singular
        assert np.allclose(X @ coef[g], X @ c, rtol=1e-7, atol=0)


def test_held_out_error_below_ten_percent(oracle):
    # 5% multiplicative noise, 500 train / 100 held out (Fig. 7 "below 10%")
    c = (0.0, 1.0, 0.0, 0.0, 3e-4)
    r = RC.make_records(5, [600], noise=0.0)
    truth = _truth(oracle, c, r["F"], r["M"])
    rng = np.random.default_rng(5)
    y = truth * (1 + 0.05 * rng.standard_normal(len(truth)))
    off = np.array([0, 500], np.int64)
    coef, _, _ = oracle.fit_perf(PERF, off, r["F"][:500], r["M"][:500], y[:500])
    pred = _pred(oracle, coef[0], r["F"][500:], r["M"][500:])
    assert np.median(np.abs(pred - truth[500:]) / truth[500:]) < 0.10


def test_intercept_only_and_constant_target(oracle):
    r = RC.make_records(6, [100])
    y = np.full(100, 0.125)
    coef, me, _ = oracle.fit_perf(PERF, r["off"], r["F"], r["M"], y)
    assert np.max(np.abs(_pred(oracle, coef[0], r["F"], r["M"]) - 0.125)) < 1e-6 * 0.125
    assert me[0] < 1e-6


def test_minimum_group_size(oracle):
    r = RC.make_records(7, [19])
    with pytest.raises(oracle.OracleError):
        oracle.fit_perf(PERF, r["off"], r["F"], r["M"], r["y"])


def test_generator_is_deterministic_and_in_range():
    a, b = RC.make_records(9, [100, 50]), RC.make_records(9, [100, 50])
    for k in ("F", "M", "y"):
        assert np.array_equal(a[k], b[k])
    assert a["M"].min() >= 10 ** 9 and a["F"].min() >= 10 ** 10 and np.all(a["y"] > 0)
    assert not np.array_equal(a["F"][:50], a["F"][100:150])  # groups draw different streams
