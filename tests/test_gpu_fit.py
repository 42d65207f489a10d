"""GPU parity of asc_fit_perf (row f2; G49) against the oracle's sequential fit.

Both sides compute bit-identical features; only the summation order of the Gram matrix differs
(chunked block reductions vs one sequential sum).  x1 = x3 + x4 makes the unregularised system
singular, so coefficients may move along that null direction with the rounding; predictions do
not.  Tolerance for predictions at the training points: 1e-8 relative (DESIGN
§Precision: Gram rounding ~1e-14 relative times the conditioning of the non-null part).
"""
import numpy as np
import pytest

from gen import presets as P
from gen import records as RC

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
PERF = P.PERF_ROOFLINE


@pytest.fixture(scope="module")
def asc():
    from paper_2504_20828_b200 import asc as A
    assert torch.cuda.is_available()
    return A


def _pred(coef, F, M):
    tM = M.astype(np.float64) / PERF["M_H"]
    tF = F.astype(np.float64) / PERF["F_H"]
    t = coef[0] * (tM + tF) + coef[1] * np.maximum(tM, tF) + coef[2] * tM + coef[3] * tF + coef[4]
    return np.maximum(t, 0.0)


def _gpu(asc, rec, lam=1e-8, host=False, errors=True):
    ctx = asc.Context(P.config(), 0)
    try:
        if host:
            return ctx.fit_perf(rec, lam, errors)
        d = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in rec.items()}
        c, me, mx = ctx.fit_perf(d, lam, errors)
        cv = lambda t: None if t is None else t.cpu().numpy()
        return cv(c), cv(me), cv(mx)
    finally:
        ctx.close()


def _check(oracle, rec, got, lam=1e-8):
    coef, me, mx = oracle.fit_perf(PERF, rec["off"], rec["F"], rec["M"], rec["y"], lam)
    gc, gme, gmx = got
    for g in range(len(rec["off"]) - 1):
        lo, hi = rec["off"][g], rec["off"][g + 1]
        pe = _pred(coef[g], rec["F"][lo:hi], rec["M"][lo:hi])
        pg = _pred(gc[g], rec["F"][lo:hi], rec["M"][lo:hi])
        # (20-record groups can extrapolate below 0: both sides clamp those predictions to 0)
        assert np.all(np.abs(pg - pe) <= 1e-8 * np.abs(pe) + 1e-18), g
    assert np.allclose(gme, me, rtol=1e-6, atol=1e-12)
    assert np.allclose(gmx, mx, rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("sizes", [[20], [8191, 8192, 8193], [20, 25, 50000, 21, 100000, 333],
                                   [20] * 3000, [24576], [8192 * 3 - 20, 40, 8192 * 2 + 7]])
def test_fit_parity(asc, oracle, sizes):
    rec = RC.make_records(11, sizes)
    _check(oracle, rec, _gpu(asc, rec))


def test_fit_round_trip_noise_free_gpu(asc, oracle):
    rec = RC.make_records(12, [5000, 300])
    for c in [(0.0, 1.0, 0.0, 0.0, 3e-4), (0.3, 0.5, 0.2, 0.1, 1e-4)]:
        pf = dict(PERF, c=c)
        y = np.array([oracle.latency_s(pf, int(f), int(m)) for f, m in zip(rec["F"], rec["M"])])
        r = dict(rec, y=y)
        gc, _, gmx = _gpu(asc, r)
        for g in range(2):
            lo, hi = r["off"][g], r["off"][g + 1]
            assert np.max(np.abs(_pred(gc[g], r["F"][lo:hi], r["M"][lo:hi]) - y[lo:hi]) / y[lo:hi]) < 1e-6
        assert np.all(gmx < 1e-6)


def test_fit_large_sampled(asc, oracle):
    # bench-sized groups (16,384 records each) over several chunks; a stratified subset of groups
    # is checked against the oracle
    sizes = [16384] * 256
    rec = RC.make_records(13, sizes)
    got = _gpu(asc, rec)
    idx = list(range(0, 256, 32))
    sub = RC.make_records(13, [0])  # structure only
    off = np.zeros(len(idx) + 1, np.int64)
    parts = []
    for j, g in enumerate(idx):
        lo, hi = rec["off"][g], rec["off"][g + 1]
        parts.append((rec["F"][lo:hi], rec["M"][lo:hi], rec["y"][lo:hi]))
        off[j + 1] = off[j] + (hi - lo)
    sub = dict(off=off, F=np.concatenate([p[0] for p in parts]), M=np.concatenate([p[1] for p in parts]),
               y=np.concatenate([p[2] for p in parts]))
    _check(oracle, sub, tuple(None if a is None else a[idx] for a in got))


def test_fit_deterministic_and_host_path(asc):
    rec = RC.make_records(14, [30000, 20, 9000])
    a = _gpu(asc, rec)
    b = _gpu(asc, rec)
    h = _gpu(asc, rec, host=True)
    for x, y_, z in zip(a, b, h):
        assert np.array_equal(x, y_) and np.array_equal(x, z)
    c, me, mx = _gpu(asc, rec, errors=False)
    assert me is None and mx is None and np.array_equal(c, a[0])


def test_fit_errors(asc):
    rec = RC.make_records(15, [100, 19])
    with pytest.raises(asc.AscError) as e:
        _gpu(asc, rec)
    assert e.value.code == 5
    rec = RC.make_records(15, [100])
    rec["y"][7] = 0.0
    with pytest.raises(asc.AscError) as e:
        _gpu(asc, rec)
    assert e.value.code == 1
    rec = RC.make_records(15, [100])
    with pytest.raises(asc.AscError) as e:
        _gpu(asc, rec, lam=-1.0)
    assert e.value.code == 1


def test_fit_unaligned_records(asc, oracle):
    # record arrays one element into their buffers (not 16-byte aligned) take fit_partials'
    # scalar-load path; the fit must not depend on it
    rec = RC.make_records(14, [20, 9000, 333, 8192])
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in rec.items()}
    for k in ("F", "M", "y"):
        big = torch.zeros(len(rec[k]) + 1, dtype=d[k].dtype, device=d[k].device)
        big[1:] = d[k]
        d[k] = big[1:]
        assert d[k].data_ptr() % 16 != 0
    ctx = asc.Context(P.config(), 0)
    try:
        c, me, mx = ctx.fit_perf(d, 1e-8, True)
        got = (c.cpu().numpy(), me.cpu().numpy(), mx.cpu().numpy())
    finally:
        ctx.close()
    _check(oracle, rec, got)
