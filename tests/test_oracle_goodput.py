"""Pins for the goodput reduction."""
import numpy as np
import pytest

from gen import traces as TR


def _batch(n, out_len, ttft=10, tbt=5):
    return TR.make_batch([(np.zeros(n, np.int64), np.ones(n), np.array(out_len))], [ttft], [tbt])


def _out(first, done, state):
    return dict(first_token_us=np.array(first, np.int64), done_us=np.array(done, np.int64),
                status=np.array(state, np.uint32))


def test_spec_examples(oracle):
    b = _batch(4, [1, 1, 1, 1])
    assert [int(x) for x in oracle.goodput(b, _out([1, 2, 3, 4], [1, 2, 3, 4], [1] * 4))[0]] == [4]
    # 3 of 4 meet TTFT -> 0.75
    g, t = oracle.goodput(b, _out([1, 2, 3, 11], [1, 2, 3, 11], [1] * 4))
    assert (int(g[0]), int(t[0])) == (3, 4)
    # TTFT met, mean TBT missed -> excluded: out 3, (done - first) = 11 > 5 * 2
    b = _batch(2, [3, 3])
    g, _ = oracle.goodput(b, _out([1, 1], [11, 12], [1, 1]))
    assert int(g[0]) == 1
    # dropped / unfinished count in the denominator only
    b = _batch(3, [1, 1, 1])
    g, t = oracle.goodput(b, _out([1, -1, -1], [1, -1, -1], [1, 2, 0]))
    assert (int(g[0]), int(t[0])) == (1, 3)


def test_empty_trace_is_an_error(oracle):
    b = TR.make_batch([(np.zeros(0), np.zeros(0), np.zeros(0))], [1], [1])
    with pytest.raises(oracle.OracleError) as e:
        oracle.goodput(b, _out([], [], []))
    assert e.value.code == 5


def test_monotone_in_slo_scale(oracle):
    # on a fixed outcome set goodput is non-decreasing in the SLO scale
    rng = np.random.default_rng(0)
    n = 500
    out_len = rng.integers(1, 50, size=n)
    first = rng.integers(0, 10 ** 6, size=n)
    done = first + rng.integers(0, 10 ** 6, size=n)
    o = _out(first, done, rng.integers(0, 3, size=n))
    prev = -1
    for k in range(1, 20):
        b = TR.make_batch([(np.zeros(n, np.int64), np.ones(n), out_len)], [k * 60_000],
                          [k * 2_000])
        g = int(oracle.goodput(b, o)[0][0])
        assert g >= prev
        prev = g
