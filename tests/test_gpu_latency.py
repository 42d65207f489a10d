"""GPU parity of asc_latency — the performance model's latency (rows a1/a6: Eq. 4-5, P:273-277,
with readings G17/G18).  SURVEY §8(c).11: "fp64 bit-exactness: GPU vs oracle t bitwise equal on
>= 10^8 random inputs" (north_star's acceptance bar is 1e-9 relative); the microseconds must be
equal too.  Inputs: (F, M) log-uniform over [1, 2^53) plus exact edge values, under four
coefficient sets (the roofline preset, mixed signs, a clamping intercept, another GPU's caps)."""
import numpy as np
import pytest

from gen import presets as P

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

PERFS = [
    P.PERF_ROOFLINE,
    dict(c=(0.1, 0.9, 0.05, -0.02, 3e-4), F_H=312e12, M_H=2e12),
    dict(c=(0.0, 0.5, 0.0, 0.0, -2e-3), F_H=312e12, M_H=2e12),      # clamps short batches to 0
    dict(c=(1.3, -0.4, 0.7, 0.2, 1e-3), F_H=2.25e15, M_H=7.7e12),
]


@pytest.fixture(scope="module")
def asc():
    from paper_2504_20828_b200 import asc as A
    assert torch.cuda.is_available()
    return A


def _inputs(rng, n):
    F = np.floor(2.0 ** rng.uniform(0.0, 53.0, n)).astype(np.uint64)
    M = np.floor(2.0 ** rng.uniform(0.0, 53.0, n)).astype(np.uint64)
    edge = np.array([0, 1, 2, 3, 10 ** 6, 2 ** 31, 2 ** 32 + 1, 2 ** 52, 2 ** 53 - 1, 312 * 10 ** 12,
                     2 * 10 ** 12, 4 * 10 ** 12 - 1], dtype=np.uint64)
    F[:len(edge)] = edge
    M[:len(edge)] = edge[::-1]
    M = np.minimum(M, np.uint64(2 ** 53 - 1))
    F = np.minimum(F, np.uint64(2 ** 53 - 1))
    return F, M


def test_latency_bitwise_1e8(asc, oracle):
    rng = np.random.default_rng(2504)
    chunk, per_perf = 5_000_000, 25_000_000          # 4 x 25M = 10^8 (F, M) pairs
    total = 0
    for pf in PERFS:
        ctx = asc.Context(P.config(perf=pf), 0)
        try:
            for _ in range(per_perf // chunk):
                F, M = _inputs(rng, chunk)
                dF = torch.from_numpy(F.view(np.int64)).cuda()
                dM = torch.from_numpy(M.view(np.int64)).cuda()
                lat, t = ctx.latency(dF, dM)
                el, et = oracle.latency_n(pf, F, M)
                got_t = t.cpu().numpy()
                bad = np.nonzero(got_t.view(np.uint64) != et.view(np.uint64))[0]
                assert len(bad) == 0, (pf, F[bad[:3]], M[bad[:3]], got_t[bad[:3]], et[bad[:3]])
                assert np.array_equal(lat.cpu().numpy(), el)
                total += chunk
        finally:
            ctx.close()
    assert total == 10 ** 8


def test_latency_host_path_and_errors(asc, oracle):
    rng = np.random.default_rng(7)
    F, M = _inputs(rng, 4096)
    ctx = asc.Context(P.config(), 0)
    try:
        lat, t = ctx.latency(F, M)                 # host arrays: staged by the library
        el, et = oracle.latency_n(P.PERF_ROOFLINE, F, M)
        assert np.array_equal(lat, el)
        assert np.array_equal(t.view(np.uint64), et.view(np.uint64))
        lat2, none = ctx.latency(F, M, want_t=False)
        assert none is None and np.array_equal(lat2, el)
        F[5] = np.uint64(2 ** 53)                  # not exactly representable: range error
        with pytest.raises(asc.AscError) as e:
            ctx.latency(F, M)
        assert e.value.code == 6
    finally:
        ctx.close()
