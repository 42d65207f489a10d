"""Edge cases of asc_simulate_batch / asc_goodput / asc_schedule_step, GPU vs oracle: empty
traces inside a batch, requests exactly at the liveness bounds (prompt + output = token budget,
KV blocks = capacity - 1), one-request traces, identical arrival times, and budgets at their
maxima (R = ASC_MAX_BATCH, N = 2^24 - 1)."""
import numpy as np
import pytest

import helpers as H
import simcases as SC
from gen import presets as P
from gen import traces as TR
from test_gpu_sim import assert_parity, gpu_sim

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def asc():
    from paper_2504_20828_b200 import asc as A
    assert torch.cuda.is_available()
    return A


def _sim_only(asc, cfg, b):
    ctx = asc.Context(cfg, 0)
    try:
        tr = asc.batch_arrays(b, "cuda:0")
        out = ctx.simulate_batch(tr)
        return {k: v.cpu().numpy() for k, v in out.items()}
    finally:
        ctx.close()


def test_empty_traces_in_a_batch(asc, oracle):
    rng = np.random.default_rng(60)
    full = SC.random_small_batch(rng, 6, 200)
    trs = []
    for t in range(6):
        trs.append(full.trace(t)[:3])
        trs.append((np.zeros(0, np.int64), np.zeros(0, np.int32), np.zeros(0, np.int32)))
    b = TR.make_batch(trs, [10 ** 6] * 12, [150_000] * 12)
    cfg = P.config()
    got = _sim_only(asc, cfg, b)
    exp = oracle.simulate_batch(cfg, b)
    for k in ("first_token_us", "done_us", "prefill_start_us"):
        assert np.array_equal(got[k][:b.R], exp[k]), k
    assert np.array_equal(got["status"][:b.R].view(np.uint32), exp["status"])
    for k in ("digest", "decisions", "evaluations"):
        assert np.array_equal(got[k][:b.T].view(exp[k].dtype), exp[k]), k
    assert np.all(got["decisions"][1:12:2] == 0)
    with pytest.raises(asc.AscError) as e:  # goodput over a trace with no requests
        ctx = asc.Context(cfg, 0)
        try:
            tr = asc.batch_arrays(b, "cuda:0")
            ctx.goodput(tr, ctx.simulate_batch(tr))
        finally:
            ctx.close()
    assert e.value.code == 5


def test_liveness_bounds(asc, oracle):
    # prompt + output == lp_token_budget and ceil((p+o)/bs) == kv_blocks - 1: the largest legal
    # requests, so evictions re-prefill prompts of exactly budget - 1 tokens
    cfg = P.config(topo=P.topology(lp_token_budget=1024, hp_token_budget=1024, block_tokens=16,
                                   kv_blocks_lp=100, kv_blocks_hp=100))
    rng = np.random.default_rng(61)
    trs = []
    for t in range(8):
        n = 60
        arr = np.cumsum(rng.integers(1, 200_000, size=n)).astype(np.int64)
        o = rng.integers(1, 500, size=n)
        p = 1024 - o
        trs.append((arr, p, o))
    b = TR.make_batch(trs, [5_000_000] * 8, [500_000] * 8)
    got = gpu_sim(asc, cfg, b)
    assert SC.npre(got["status"]).sum() > 0  # evictions of maximal requests happen
    assert_parity(oracle, cfg, b, got)
    bad = TR.make_batch([(np.array([0], np.int64), np.array([1000]), np.array([25]))], [10 ** 6], [10 ** 5])
    with pytest.raises(asc.AscError) as e:  # prompt + output = 1025 > budget
        gpu_sim(asc, cfg, bad)
    assert e.value.code == 2


def test_identical_arrivals_and_singletons(asc, oracle):
    rng = np.random.default_rng(62)
    trs = []
    for t in range(40):
        n = 1 if t % 2 else 50
        arr = np.full(n, 1_000_000 * (t % 3), np.int64)  # every request of a trace at once
        trs.append((arr, rng.integers(4, 2000, size=n), rng.integers(1, 300, size=n)))
    b = TR.make_batch(trs, [10 ** 6] * 40, [150_000] * 40)
    for pol in ("EDF_LAXITY", "SJF", "FCFS"):
        cfg = P.config(flg=P.flags(policy=pol, drop=1))
        assert_parity(oracle, cfg, b, gpu_sim(asc, cfg, b))


def test_step_budget_maxima(asc, oracle):
    from test_gpu_step import compare, run_gpu
    rng = np.random.default_rng(63)
    # (the ctx's lp_token_budget sizes the prefill table: F of a 16M-token prompt would pass 2^53,
    # which asc_create rejects with ASC_E_RANGE; the per-segment budgets are the maxima here)
    cfg = P.config(topo=P.topology(lp_max_batch=128, lp_token_budget=65536))
    ins = H.random_step_inputs(rng, 40, 0, cfg, qs=np.full(40, 300))
    ins["budget_reqs"][:] = 128
    ins["budget_tokens"][:] = (1 << 24) - 1
    ins["budget_blocks"][:] = (1 << 22) - 1
    compare(run_gpu(asc, cfg, ins), oracle.schedule_step(cfg, **ins), ins["seg_off"])


@pytest.mark.parametrize("elastic", [0, 1])
def test_hp_decode_set_beyond_shared_slots(asc, oracle, elastic):
    # an offload margin of 10^6 s sends every request the LP does not admit to the HP, whose
    # prefill batches then leave ~900 concurrent decodes: slots beyond the 128 kept in shared memory
    # live in HBM (sim.cu DCAP), through decode runs and completions alike
    cfg = P.config(topo=P.topology(n_lp=1, n_hp=1), flg=P.flags(offload_margin_us=10 ** 12, elastic=elastic))
    n = 1200
    arr = np.zeros(n, np.int64)
    arr[600:] = 5_000_000
    b = TR.make_batch([(arr, np.full(n, 16, np.int32), np.full(n, 300, np.int32))], [10 ** 9], [10 ** 9])
    got = gpu_sim(asc, cfg, b)
    st = got["status"]
    hp = ((st >> 4) & 0xff) == 1
    assert hp.sum() > 500
    assert_parity(oracle, cfg, b, got)


def test_step_range_errors(asc, oracle):
    # eff_prompt >= 2^24 and a dec_ctx_sum whose uint64 decode cost would wrap are
    # ASC_E_RANGE on both sides (the oracle rejects the first; the second is a GPU-side guard)
    from test_gpu_step import run_gpu
    cfg = P.config()
    rng = np.random.default_rng(64)
    for case in ("eff", "ctx"):
        ins = H.random_step_inputs(rng, 6, 0, cfg, qs=np.array([0, 1, 40, 33, 5000, 20000]))
        if case == "eff":
            ins["eff_prompt"][-3] = 1 << 24
        else:
            ins["dec_count"][3] = 100
            ins["dec_ctx_sum"][3] = 1 << 62
        with pytest.raises(asc.AscError) as e:
            run_gpu(asc, cfg, ins)
        assert e.value.code == 6
        if case == "eff":
            with pytest.raises(oracle.OracleError) as e2:
                oracle.schedule_step(cfg, **ins)
            assert e2.value.code == 6


def test_small_segment_packed_sort_window_edge(asc, oracle):
    # k_small packs (key - now + 2^26) << 5 | lane into 32 bits; a key of exactly
    # now + 2^26 - 1 in lane 31 must not collide with the dead-lane sentinel 0xffffffff
    from test_gpu_step import compare, run_gpu
    cfg = P.config(flg=P.flags(policy="EDF_DEADLINE"))  # key = deadline
    S = 4
    ins = H.random_step_inputs(np.random.default_rng(65), S, 0, cfg, qs=np.full(S, 32), budgets="max")
    for s in range(S):
        lo = 32 * s
        ins["deadline_us"][lo:lo + 32] = ins["now_us"][s] + np.arange(32) * 1000 + 10 ** 6
        ins["deadline_us"][lo + 31] = ins["now_us"][s] + (1 << 26) - 1 - s  # s = 0: the edge
        ins["eff_prompt"][lo:lo + 32] = 10
        ins["flags"][lo:lo + 32] = 0
    ins["dec_count"][:] = 0
    exp = oracle.schedule_step(cfg, **ins)
    assert all(int(c) == 32 for c in exp["admit_cnt"])
    compare(run_gpu(asc, cfg, ins), exp, ins["seg_off"])


def test_decode_context_sum_below_count_is_inval(asc, oracle):
    # every decode context lhat >= 1, so dec_ctx_sum >= dec_count (oracle: "dec_ctx_sum < dec_count");
    # dec_ctx_sum is ignored when dec_count = 0 (test above)
    from test_gpu_step import run_gpu
    cfg = P.config()
    for qs in (np.array([0, 20, 30]), np.array([0, 20, 20000])):   # k_small and k1 segments
        ins = H.random_step_inputs(np.random.default_rng(66), 3, 0, cfg, qs=qs)
        ins["dec_count"][2] = 5
        ins["dec_ctx_sum"][2] = 4
        with pytest.raises(asc.AscError) as e:
            run_gpu(asc, cfg, ins)
        assert e.value.code == 1
        with pytest.raises(oracle.OracleError) as e2:
            oracle.schedule_step(cfg, **ins)
        assert e2.value.code == 1
