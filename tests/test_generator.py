"""The seeded input generator (gen/): determinism, counter recipe, distribution shape."""
import numpy as np

from gen import presets as P
from gen import traces as TR


def test_splitmix_known_values():
    # splitmix64 finalizer reference values computed with Python integers
    assert TR.mix_int(0) == 0
    x = np.array([0, 1, 2 ** 63, 12345], np.uint64)
    assert [int(v) for v in TR.mix_np(x)] == [TR.mix_int(int(v)) for v in x]


def test_counter_recipe():
    a, p, o = TR.gen_trace(7, 3, "sharegpt", 16, 50)
    seed = TR.mix_int(7 ^ 3)
    t = TR.tables()
    for i in (0, 17, 49):
        u1 = TR.mix_int(seed + (3 * i + 1) * TR.GOLDEN)
        u2 = TR.mix_int(seed + (3 * i + 2) * TR.GOLDEN)
        assert p[i] == t["sharegpt_prompt"][u1 >> 48]
        assert o[i] == t["sharegpt_output"][u2 >> 48]
    gaps = np.diff(np.concatenate([[0], a]))
    u0 = TR.mix_int(seed + 0)
    assert gaps[0] == (int(t["exp_q32"][u0 >> 48]) * 8_000_000 // 16) >> 32


def test_shapes_and_rates():
    a, p, o = TR.gen_trace(1, 0, "sharegpt", 16, 20000)     # QPS 2
    assert np.all(np.diff(a) >= 0)
    assert abs(a[-1] / 1e6 / 20000 - 0.5) < 0.02            # mean gap 0.5 s (Poisson)
    assert 4 <= p.min() and p.max() <= 4096 and 1 <= o.min() and o.max() <= 2048
    assert 200 < np.median(p) < 300                          # lognormal(5.5, 1) median ~245
    a, p, o = TR.gen_trace(1, 0, "longbench", 8, 5000)
    assert 512 <= p.min() and p.max() <= 32768 and 16 <= o.min() and o.max() <= 512


def test_workloads_valid():
    for w in ("config1", "config2", "config3", "config4", "config5"):
        cfg, b = P.workload(w, n=50, max_traces=20)
        t = cfg["topo"]
        assert np.all(b.prompt_len.astype(np.int64) + b.output_len <= t["lp_token_budget"])
    cfg, b = P.workload("config3", n=10)
    assert b.T == 4096 and len(set(zip(b.qps_j, b.ttft_slo_us))) == 256


def test_select_generates_a_shard_alone():
    """workload(select=) (bench.py's config-5 shards) equals subsetting the full grid."""
    from paper_2504_20828_b200 import dist as D
    cfg, full = P.workload("config5", n=40, max_traces=64)
    for r, W in ((0, 4), (3, 4), (1, 7)):
        idx = D.shard(full.T, r, W)
        _, sub = P.workload("config5", n=40, max_traces=64, select=idx)
        ref = full.subset(idx)
        for k in ("trace_off", "arrival_us", "prompt_len", "output_len", "ttft_slo_us", "tbt_slo_us", "qps_j"):
            assert np.array_equal(getattr(sub, k), getattr(ref, k)), k
        assert sub.labels == ref.labels
