"""GPU parity of asc_schedule_step (rows a1-a6) against the oracle, through the C ABI.

Integer outputs (admission lists in priority order, offload/drop lists, counts, microsecond
latencies) must be bit-exact; prefill latencies are compared exactly (the fp64 op order is fixed,
DESIGN.md §Bit-exactness), which is stricter than north_star's 1e-9 relative bound.
"""
import numpy as np
import pytest

import helpers as H
from gen import presets as P

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def asc():
    from paper_2504_20828_b200 import asc as A
    assert torch.cuda.is_available()
    return A


def to_dev(ins):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in ins.items()}


def run_gpu(asc, cfg, ins, host=False):
    ctx = asc.Context(cfg, 0)
    try:
        if host:
            out = ctx.schedule_step({k: np.ascontiguousarray(v) for k, v in ins.items()})
        else:
            out = ctx.schedule_step(to_dev(ins))
            out = {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}
        launches = ctx.last_launches()
    finally:
        ctx.close()
    assert launches >= 1
    return out


def compare(got, exp, seg_off):
    S = len(seg_off) - 1
    Q = int(seg_off[-1])
    for k in ("admit_cnt", "offload_cnt", "drop_cnt", "batch_lat_us"):
        assert np.array_equal(got[k][:S], exp[k][:S]), k
    assert np.array_equal(got["prefill_us"][:Q], exp["prefill_us"][:Q])
    g = H.segment_lists(got, seg_off)
    e = H.segment_lists(exp, seg_off)
    for s in range(S):
        assert g[s] == e[s], f"segment {s}"


@pytest.mark.parametrize("policy", ["EDF_LAXITY", "EDF_DEADLINE", "FCFS", "SJF", "LJF"])
def test_w1_hand_worked_gpu(asc, policy):
    cfg, ins, exp, rid = H.w1_step_inputs(policy)
    out = run_gpu(asc, cfg, ins)
    adm, off, drp = H.segment_lists(out, ins["seg_off"])[0]
    assert [rid[i] for i in adm] == exp["admitted"]
    assert [rid[i] for i in off] == exp["offloaded"]
    assert out["batch_lat_us"][0] == exp["batch_lat"] * H.SEC


def test_prefill_table_exhaustive(asc, oracle):
    # a1 for every prompt length the LongBench preset can produce, and beyond the table
    cfg = P.config(topo=P.topology(lp_token_budget=65536))
    Q = 70000
    ins = dict(seg_off=np.array([0, Q], np.int64), now_us=np.zeros(1, np.int64),
               deadline_us=np.full(Q, 10 ** 12, np.int64),
               eff_prompt=np.arange(1, Q + 1, dtype=np.int32), flags=np.zeros(Q, np.uint8),
               dec_count=np.zeros(1, np.int32), dec_ctx_sum=np.zeros(1, np.int64),
               tbt_slo_us=np.zeros(1, np.int64), budget_tokens=np.zeros(1, np.int32),
               budget_blocks=np.zeros(1, np.int32), budget_reqs=np.zeros(1, np.int32))
    got = run_gpu(asc, cfg, ins)
    exp = oracle.schedule_step(cfg, **ins)
    assert np.array_equal(got["prefill_us"][:Q], exp["prefill_us"])


@pytest.mark.parametrize("policy", ["EDF_LAXITY", "EDF_DEADLINE", "FCFS", "SJF", "LJF"])
@pytest.mark.parametrize("drop", [0, 1])
def test_random_segments_shallow(asc, oracle, policy, drop):
    rng = np.random.default_rng(hash((policy, drop)) % 2 ** 32)
    cfg = P.config(flg=P.flags(policy=policy, drop=drop))
    ins = H.random_step_inputs(rng, 300, 60, cfg)
    compare(run_gpu(asc, cfg, ins), oracle.schedule_step(cfg, **ins), ins["seg_off"])


@pytest.mark.parametrize("policy", ["EDF_LAXITY", "SJF", "FCFS", "LJF"])
def test_random_segments_multi_task(asc, oracle, policy):
    # segments spanning several 2048-entry warp tasks plus a ragged tail, and empty segments
    rng = np.random.default_rng(7)
    cfg = P.config(flg=P.flags(policy=policy, drop=1))
    qs = [0, 1, 2047, 2048, 2049, 6000, 0, 13000, 31, 4097]
    ins = H.random_step_inputs(rng, len(qs), 0, cfg, qs=qs)
    compare(run_gpu(asc, cfg, ins), oracle.schedule_step(cfg, **ins), ins["seg_off"])


def test_deep_segments_ample_budgets(asc, oracle):
    rng = np.random.default_rng(9)
    cfg = P.config()
    ins = H.random_step_inputs(rng, 4, 0, cfg, budgets="config", qs=[100_000, 50_000, 3, 70_001])
    compare(run_gpu(asc, cfg, ins), oracle.schedule_step(cfg, **ins), ins["seg_off"])


@pytest.mark.parametrize("bind", ["tokens", "blocks", "tbt", "reqs", "mixed"])
def test_budget_bound_thresholds(asc, oracle, bind):
    # k1 moves its selection threshold to the first list position whose running tokens / blocks /
    # prefill µs reach N / M / C (Alg. 1 l.5-13): deep single- and multi-task segments
    # where each budget binds in turn, with heavily tied keys (deadlines on a coarse grid)
    rng = np.random.default_rng({"tokens": 11, "blocks": 12, "tbt": 13, "reqs": 14, "mixed": 15}[bind])
    cfg = P.config(flg=P.flags(policy="EDF_LAXITY", drop=1))
    qs = [16384, 16385, 40000, 9000, 33, 70000, 12000, 5000]
    ins = H.random_step_inputs(rng, len(qs), 0, cfg, budgets="config", qs=qs)
    S = len(qs)
    ins["deadline_us"] = (ins["deadline_us"] // 250_000) * 250_000
    if bind in ("tokens", "mixed"):
        ins["budget_tokens"] = rng.integers(1, 3000, size=S).astype(np.int32)
    if bind in ("blocks", "mixed"):
        ins["budget_blocks"] = rng.integers(1, 120, size=S).astype(np.int32)
    if bind in ("tbt", "mixed"):
        ins["dec_count"] = rng.integers(1, 64, size=S).astype(np.int32)
        ins["dec_ctx_sum"] = ins["dec_count"].astype(np.int64) * 500
        ins["tbt_slo_us"] = rng.integers(20_000, 300_000, size=S).astype(np.int64)
    if bind == "reqs":
        ins["budget_reqs"] = rng.integers(1, 129, size=S).astype(np.int32)
    got = run_gpu(asc, cfg, ins)
    exp = oracle.schedule_step(cfg, **ins)
    assert int(exp["admit_cnt"].sum()) > 0
    compare(got, exp, ins["seg_off"])


def test_adversarial_key_order(asc, oracle):
    # keys strictly decreasing with position: every entry beats the running threshold
    cfg = P.config(flg=P.flags(policy="EDF_DEADLINE"))
    Q = 9000
    ins = dict(seg_off=np.array([0, Q], np.int64), now_us=np.array([10 ** 7], np.int64),
               deadline_us=(2 * 10 ** 7 - np.arange(Q, dtype=np.int64) * 7),
               eff_prompt=np.full(Q, 50, np.int32), flags=np.zeros(Q, np.uint8),
               dec_count=np.zeros(1, np.int32), dec_ctx_sum=np.zeros(1, np.int64),
               tbt_slo_us=np.zeros(1, np.int64), budget_tokens=np.array([8192], np.int32),
               budget_blocks=np.array([25000], np.int32), budget_reqs=np.array([128], np.int32))
    compare(run_gpu(asc, cfg, ins), oracle.schedule_step(cfg, **ins), ins["seg_off"])


def test_host_pointer_path(asc, oracle):
    rng = np.random.default_rng(3)
    cfg = P.config(flg=P.flags(drop=1))
    ins = H.random_step_inputs(rng, 50, 3000, cfg)
    got = run_gpu(asc, cfg, ins, host=True)
    compare(got, oracle.schedule_step(cfg, **ins), ins["seg_off"])


def test_host_pointer_path_many_segments(asc, oracle):
    # S >= 4096 with prefill_us requested: the staging buffer must hold all seven [S] int32
    # arrays (the size formula counted five, so the last staged array overran it)
    rng = np.random.default_rng(33)
    cfg = P.config(flg=P.flags(drop=1))
    ins = H.random_step_inputs(rng, 6000, 0, cfg, qs=rng.integers(0, 40, size=6000))
    got = run_gpu(asc, cfg, ins, host=True)
    compare(got, oracle.schedule_step(cfg, **ins), ins["seg_off"])


def test_many_tiny_segments(asc, oracle):
    rng = np.random.default_rng(4)
    cfg = P.config()
    ins = H.random_step_inputs(rng, 20000, 0, cfg, qs=np.full(20000, 32))
    compare(run_gpu(asc, cfg, ins), oracle.schedule_step(cfg, **ins), ins["seg_off"])


@pytest.mark.parametrize("spread_us", [3 * 10 ** 6, 10 ** 9, 10 ** 11])
@pytest.mark.parametrize("policy", ["EDF_LAXITY", "FCFS", "SJF"])
def test_small_segment_key_windows(asc, oracle, spread_us, policy):
    # k_small sorts (key - now, position) packed in 32 bits when every key lies within 2^26 us of
    # now, in 64 bits within 2^31 us, else as (int64 key, position): all three must agree
    rng = np.random.default_rng(31)
    cfg = P.config(flg=P.flags(policy=policy, drop=1))
    qs = rng.integers(0, 33, size=3000)
    ins = H.random_step_inputs(rng, 3000, 0, cfg, qs=qs, now_spread_us=spread_us)
    compare(run_gpu(asc, cfg, ins), oracle.schedule_step(cfg, **ins), ins["seg_off"])


def test_many_segments_mixed_sizes(asc, oracle):
    # S > 8191 takes the multi-launch planner (count, tile scans, task map); segments of every
    # kind in one call: short (k_small), single-task (k1), multi-task (k1 + k2 + k3)
    rng = np.random.default_rng(41)
    S = 12000
    qs = rng.integers(0, 33, size=S)
    mid = rng.random(S) < 0.25
    qs[mid] = rng.integers(33, 1500, size=int(mid.sum()))
    qs[[17, 5000, 11999]] = [40000, 16385, 33000]
    cfg = P.config()
    ins = H.random_step_inputs(rng, S, 0, cfg, qs=qs)
    compare(run_gpu(asc, cfg, ins), oracle.schedule_step(cfg, **ins), ins["seg_off"])


def test_unaligned_inputs(asc, oracle):
    # per-entry arrays that are not 16-byte aligned (views one element into a buffer) take k1's
    # scalar-load path (VEC = false) and k_small's; results must not depend on it
    rng = np.random.default_rng(43)
    cfg = P.config(flg=P.flags(drop=1))
    qs = rng.integers(0, 33, size=600)
    qs[::7] = rng.integers(33, 3000, size=len(qs[::7]))
    qs[5] = 20000
    ins = H.random_step_inputs(rng, 600, 0, cfg, qs=qs)
    d = to_dev(ins)
    for k in ("deadline_us", "eff_prompt", "flags"):
        big = torch.zeros(len(ins[k]) + 1, dtype=d[k].dtype, device=d[k].device)
        big[1:] = d[k]
        d[k] = big[1:]
        assert d[k].data_ptr() % 16 != 0
    ctx = asc.Context(cfg, 0)
    try:
        out = ctx.schedule_step(d)
        out = {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}
    finally:
        ctx.close()
    compare(out, oracle.schedule_step(cfg, **ins), ins["seg_off"])


def test_errors(asc):
    rng = np.random.default_rng(5)
    cfg = P.config()
    ins = H.random_step_inputs(rng, 3, 10, cfg)
    bad = dict(ins, budget_reqs=np.array([129, 1, 1], np.int32))
    with pytest.raises(asc.AscError) as e:
        run_gpu(asc, cfg, bad)
    assert e.value.code == 6
    ins2 = H.random_step_inputs(rng, 2, 0, cfg, qs=[3, 3])
    ins2["eff_prompt"][1] = 0
    with pytest.raises(asc.AscError) as e:
        run_gpu(asc, cfg, ins2)
    assert e.value.code == 1


def test_generic_path_wide_deadlines(asc, oracle):
    # deadlines hours away from `now` leave the 32-bit fast-path window: the exact 64-bit path
    # must take over for those tasks (mixed with in-window segments)
    rng = np.random.default_rng(21)
    for pol in ("EDF_LAXITY", "SJF"):
        cfg = P.config(flg=P.flags(policy=pol, drop=1))
        ins = H.random_step_inputs(rng, 6, 0, cfg, qs=[300, 5000, 40000, 7, 0, 20000])
        ins["deadline_us"][:300] += 10 ** 12
        ins["deadline_us"][5300:5400] -= 5 * 10 ** 10
        compare(run_gpu(asc, cfg, ins), oracle.schedule_step(cfg, **ins), ins["seg_off"])


def test_row_s_full_scale_sampled(asc, oracle):
    """SURVEY row S at full size (4096 segments x 10,000 entries) with bench.py's inputs and launch
    configuration; the oracle checks a stratified sample of segments one by one (segments are
    independent, so a segment's decision depends only on its own entries and budgets)."""
    rng = np.random.default_rng(123)  # bench.py's step_microbench seed
    cfg = P.config()
    S, Qs = 4096, 10_000
    ins = H.random_step_inputs(rng, S, 0, cfg, qs=np.full(S, Qs))
    got = run_gpu(asc, cfg, ins)
    g = H.segment_lists(got, ins["seg_off"])
    for s in range(0, S, 128):
        lo, hi = int(ins["seg_off"][s]), int(ins["seg_off"][s + 1])
        one = dict(seg_off=np.array([0, hi - lo], np.int64))
        for k in ("now_us", "dec_count", "dec_ctx_sum", "tbt_slo_us", "budget_tokens", "budget_blocks",
                  "budget_reqs"):
            one[k] = ins[k][s:s + 1]
        for k in ("deadline_us", "eff_prompt", "flags"):
            one[k] = ins[k][lo:hi]
        exp = oracle.schedule_step(cfg, **one)
        e = H.segment_lists(exp, one["seg_off"])[0]
        assert [list(np.asarray(x) - lo) for x in g[s]] == [list(x) for x in e], s
        assert got["batch_lat_us"][s] == exp["batch_lat_us"][0], s


def compare_vec(got, exp, seg_off):
    """compare() without per-segment Python lists (millions of segments): counts and latencies
    element by element, then every list slot below its segment's count."""
    S = len(seg_off) - 1
    Q = int(seg_off[-1])
    for k in ("admit_cnt", "offload_cnt", "drop_cnt", "batch_lat_us"):
        assert np.array_equal(got[k][:S], exp[k][:S]), k
    seg_of = np.repeat(np.arange(S), np.diff(seg_off))
    local = np.arange(Q) - seg_off[:-1][seg_of]
    for idx, cnt in (("admit_idx", "admit_cnt"), ("offload_idx", "offload_cnt"), ("drop_idx", "drop_cnt")):
        m = local < exp[cnt][seg_of]
        bad = np.flatnonzero(got[idx][:Q][m] != exp[idx][:Q][m])
        assert bad.size == 0, (idx, int(seg_of[np.flatnonzero(m)[bad[0]]]))


def test_row_s_short_queues_full_scale(asc, oracle):
    """SURVEY row S's third shape at full size, bench.py's inputs (10^6 segments x 32 entries,
    seed 123): k_lane decides every segment one per thread; the whole call equals the oracle."""
    rng = np.random.default_rng(123)
    cfg = P.config()
    S = 1_000_000
    ins = H.random_step_inputs(rng, S, 0, cfg, qs=np.full(S, 32))
    got = run_gpu(asc, cfg, ins)
    compare_vec(got, oracle.schedule_step(cfg, **ins), ins["seg_off"])


@pytest.mark.parametrize("policy", ["EDF_LAXITY", "EDF_DEADLINE", "FCFS", "SJF", "LJF"])
def test_lane_handback_mix(asc, oracle, policy):
    """Groups of 32 short segments where some segments leave k_lane's fast window and are handed
    to k_small: prompts beyond the 2^17-entry fast table, keys more than 2^26 us from now (both
    directions), no decodes, zero budgets, empty segments; plus groups that contain a k1 segment
    (the group's entry range exceeds the staging buffer)."""
    rng = np.random.default_rng(77)
    cfg = P.config(flg=P.flags(policy=policy, drop=1))
    S = 4000
    qs = rng.integers(0, 33, size=S)
    qs[::211] = 200
    ins = H.random_step_inputs(rng, S, 0, cfg, qs=qs)
    off = ins["seg_off"]
    for s in rng.choice(S, 300, replace=False):
        lo, hi = int(off[s]), int(off[s + 1])
        if hi == lo:
            continue
        j = int(rng.integers(lo, hi))
        kind = s % 4
        if kind == 0:
            ins["eff_prompt"][j] = int(rng.integers((1 << 17) + 1, (1 << 17) + 5000))
        elif kind == 1:
            ins["deadline_us"][j] += (1 << 27)
        elif kind == 2:
            ins["deadline_us"][j] -= (1 << 27)
        else:
            ins["deadline_us"][j] = ins["now_us"][s] + (1 << 26) - 2
    z = rng.random(S) < 0.1
    ins["dec_count"][z] = 0
    ins["budget_tokens"][rng.random(S) < 0.02] = 0
    ins["budget_reqs"][rng.random(S) < 0.02] = 0
    compare(run_gpu(asc, cfg, ins), oracle.schedule_step(cfg, **ins), ins["seg_off"])


@pytest.mark.slow
def test_row_s_deep_segments_full_scale(asc, oracle):
    """SURVEY row S's second shape at full size, bench.py's inputs (64 segments x 10^6 entries,
    seed 123): multi-task segments through k1, the k2 merge and the k3 expansion; every slot of
    every list equals the oracle."""
    rng = np.random.default_rng(123)
    cfg = P.config()
    S = 64
    ins = H.random_step_inputs(rng, S, 0, cfg, qs=np.full(S, 1_000_000))
    got = run_gpu(asc, cfg, ins)
    compare_vec(got, oracle.schedule_step(cfg, **ins), ins["seg_off"])
