"""Pins for the outcome summary (row a8): P:579-584 (Fig. 10: P99 TTFT, mean TBT, throughput,
scheduling delay per instance type), SPEC S:543-590 (metrics module: nearest-rank percentiles
S:567-573, counts, tokens, HP-path delay reported apart from LP-path S:583), DESIGN reading G52."""
import numpy as np

from gen import presets as P
from gen import traces as TR

CFG = P.config(topo=P.topology(n_lp=2, n_hp=1))


def _batch(arrival, out_len, ttft=10, tbt=5):
    n = len(arrival)
    return TR.make_batch([(np.array(arrival, np.int64), np.ones(n), np.array(out_len))], [ttft], [tbt])


def _out(first, done, pstart, state, inst=None):
    n = len(first)
    inst = np.zeros(n, np.uint32) if inst is None else np.array(inst, np.uint32)
    return dict(first_token_us=np.array(first, np.int64), done_us=np.array(done, np.int64),
                prefill_start_us=np.array(pstart, np.int64),
                status=np.array(state, np.uint32) | (inst << 4))


def test_nearest_rank_spec_examples(oracle):
    # [1..100], q = 99 -> 99 (and q = 50 -> 50, q = 90 -> 90 by the same definition)
    n = 100
    b = _batch(np.zeros(n), np.ones(n))
    f = np.arange(1, n + 1)
    s = oracle.summarize(CFG, b, _out(f[::-1], f[::-1], np.zeros(n), np.ones(n)))
    assert (int(s["ttft_p50_us"][0]), int(s["ttft_p90_us"][0]), int(s["ttft_p99_us"][0])) == (50, 90, 99)
    # a single value -> that value for every q
    b = _batch([3], [1])
    s = oracle.summarize(CFG, b, _out([10], [10], [4], [1]))
    assert (int(s["ttft_p50_us"][0]), int(s["ttft_p99_us"][0])) == (7, 7)


def test_percentiles_match_inverted_cdf(oracle):
    # nearest rank = the smallest x with empirical CDF >= q: numpy's "inverted_cdf" method
    rng = np.random.default_rng(5)
    for n in (1, 2, 7, 99, 100, 101, 1000, 4321):
        arr = np.sort(rng.integers(0, 10 ** 6, size=n))
        first = arr + rng.integers(0, 10 ** 7, size=n)
        has = rng.random(n) < 0.9
        first = np.where(has, first, -1)
        b = _batch(arr, np.ones(n))
        s = oracle.summarize(CFG, b, _out(first, first, first, np.where(has, 1, 0)))
        v = (first - arr)[has]
        for q, k in ((50, "ttft_p50_us"), (90, "ttft_p90_us"), (99, "ttft_p99_us")):
            exp = int(np.percentile(v, q, method="inverted_cdf")) if len(v) else -1
            assert int(s[k][0]) == exp, (n, q)


def test_counts_tokens_tbt_and_delay_split(oracle):
    # hand-built trace: 5 requests, instance 2 is the HP of a 2L1H trace
    arrival = [0, 0, 5, 10, 20]
    out_len = [1, 3, 2, 4, 5]
    first = [6, 8, 9, -1, 40]
    done = [6, 30, 12, -1, 60]
    pstart = [1, 2, 7, -1, 25]
    state = [1, 1, 1, 2, 0]          # completed x3, dropped, unfinished
    inst = [0, 2, 1, 255, 2]
    b = _batch(arrival, out_len, ttft=6, tbt=5)
    s = oracle.summarize(CFG, b, _out(first, done, pstart, state, inst))
    assert int(s["completed"][0]) == 3 and int(s["dropped"][0]) == 1
    # good: r0 (ttft 6 <= 6, out 1), r2 (ttft 4, tbt 3 <= 5); r1 misses TTFT (8 > 6)
    assert int(s["violating"][0]) == 1
    assert int(s["tokens"][0]) == 1 + 3 + 2
    assert int(s["tbt_sum_us"][0]) == (30 - 8) + (12 - 9) and int(s["tbt_tokens"][0]) == 2 + 1
    # LP (instances 0, 1): r0 delay 1, r2 delay 2; HP (instance 2): r1 delay 2, r4 delay 5
    assert (int(s["delay_sum_lp_us"][0]), int(s["delay_cnt_lp"][0])) == (3, 2)
    assert (int(s["delay_sum_hp_us"][0]), int(s["delay_cnt_hp"][0])) == (7, 2)
    assert int(s["last_done_us"][0]) == 30
    # with a per-trace topology of 1 LP, instance 1 counts as HP
    s1 = oracle.summarize(CFG, b, _out(first, done, pstart, state, inst), n_lp=[1])
    assert (int(s1["delay_cnt_lp"][0]), int(s1["delay_cnt_hp"][0])) == (1, 3)
    # S:589 throughput example arithmetic: 100 requests x 200 tokens over a 100 s window
    n = 100
    b = _batch(np.zeros(n), np.full(n, 200), ttft=10 ** 9, tbt=10 ** 9)
    s = oracle.summarize(CFG, b, _out(np.zeros(n), np.full(n, 100 * 10 ** 6), np.zeros(n), np.ones(n)))
    assert int(s["tokens"][0]) / ((int(s["last_done_us"][0]) - 0) / 1e6) == 200.0


def test_summary_consistent_with_goodput_and_simulation(oracle):
    # invariants on real simulated traces: completed + dropped + unfinished = total,
    # good = completed - violating, every request with a prefill start is counted once
    cfg, b = P.workload("config3", n=400, max_traces=12)
    out = oracle.simulate_batch(cfg, b, nthreads=4)
    g, t = oracle.goodput(b, out)
    s = oracle.summarize(cfg, b, out)
    st = out["status"] & 3
    for i in range(b.T):
        a, e = int(b.trace_off[i]), int(b.trace_off[i + 1])
        assert int(s["completed"][i]) + int(s["dropped"][i]) + int((st[a:e] == 0).sum()) == int(t[i])
        assert int(s["completed"][i]) - int(s["violating"][i]) == int(g[i])
        assert int(s["delay_cnt_lp"][i] + s["delay_cnt_hp"][i]) == int((out["prefill_start_us"][a:e] >= 0).sum())
