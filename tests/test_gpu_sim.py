"""GPU parity of asc_simulate_batch (row a7 with a1-a6 inlined) and asc_goodput (row a8).

Per-request event times (integer microseconds), status words, per-trace schedule digests,
decision and evaluation counts must equal the oracle's bit for bit; the hand-stepped traces
W2-W5 and the closed forms pin the GPU path directly as well.
"""
import numpy as np
import pytest

import helpers as H
import simcases as SC
from gen import presets as P
from gen import traces as TR

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def asc():
    from paper_2504_20828_b200 import asc as A
    assert torch.cuda.is_available()
    return A


def gpu_sim(asc, cfg, batch, rt=None, host=False):
    ctx = asc.Context(cfg, 0)
    try:
        if host:
            tr = asc.batch_arrays(batch)
            out = ctx.simulate_batch(tr, req_ttft_slo_us=rt)
            good, total = ctx.goodput(tr, out, req_ttft_slo_us=rt)
        else:
            tr = asc.batch_arrays(batch, "cuda:0")
            drt = None if rt is None else torch.from_numpy(np.ascontiguousarray(rt)).cuda()
            out = ctx.simulate_batch(tr, req_ttft_slo_us=drt)
            good, total = ctx.goodput(tr, out, req_ttft_slo_us=drt)
            out = {k: v.cpu().numpy() for k, v in out.items()}
            good, total = good.cpu().numpy(), total.cpu().numpy()
    finally:
        ctx.close()
    R, T = batch.R, batch.T
    res = {k: out[k][:R] for k in ("first_token_us", "done_us", "prefill_start_us")}
    res["status"] = out["status"][:R].view(np.uint32)
    res["digest"] = out["digest"][:T].view(np.uint64)
    res["decisions"] = out["decisions"][:T]
    res["evaluations"] = out["evaluations"][:T]
    res["good"] = good[:T].view(np.uint64)
    res["total"] = total[:T].view(np.uint64)
    return res


def assert_parity(oracle, cfg, batch, got, rt=None):
    exp = oracle.simulate_batch(cfg, batch, req_ttft_slo_us=rt)
    for k in ("first_token_us", "done_us", "prefill_start_us", "status"):
        bad = np.nonzero(got[k] != exp[k])[0]
        assert len(bad) == 0, f"{k}: first mismatch at request {bad[:5]}: {got[k][bad[:5]]} vs {exp[k][bad[:5]]}"
    for k in ("digest", "decisions", "evaluations"):
        assert np.array_equal(got[k], exp[k]), k
    g, t = oracle.goodput(batch, exp, req_ttft_slo_us=rt)
    assert np.array_equal(got["good"], g) and np.array_equal(got["total"], t)


@pytest.mark.parametrize("name", ["w2_two_request_des.json", "w3_tickets_offload.json",
                                  "w4_preemption.json"])
def test_hand_stepped_gpu(asc, name):
    sim = lambda cfg, b, rt=None: gpu_sim(asc, cfg, b, rt)
    gp = lambda b, o: (o["good"], o["total"])
    SC.check_fixture(sim, gp, name)


def test_elastic_gpu(asc):
    SC.check_elastic(lambda cfg, b, rt=None: gpu_sim(asc, cfg, b, rt))


def test_lindley_and_closed_forms_gpu(asc):
    rng = np.random.default_rng(1)
    for n in (1, 7, 300):
        cfg, b, end = SC.lindley_case(rng, n)
        assert [int(x) for x in gpu_sim(asc, cfg, b)["first_token_us"]] == end
    for p, o in [(1, 1), (17, 40), (300, 7)]:
        cfg, b, first, done = SC.single_request_case(p, o)
        r = gpu_sim(asc, cfg, b)
        assert int(r["first_token_us"][0]) == first and int(r["done_us"][0]) == done


def test_textbook_rules_gpu(asc):
    SC.check_textbook_rules(lambda cfg, b, rt=None: gpu_sim(asc, cfg, b, rt),
                            lambda b, o: (o["good"], o["total"]), np.random.default_rng(2), trials=15)


def test_config1_full(asc, oracle):
    cfg, b = P.workload("config1")
    assert_parity(oracle, cfg, b, gpu_sim(asc, cfg, b))


def test_config2_reduced(asc, oracle):
    cfg, b = P.workload("config2", n=2000)
    assert_parity(oracle, cfg, b, gpu_sim(asc, cfg, b))


def test_config2_full(asc, oracle):
    # BASELINE config 2 at its full size: 8 traces (QPS 1..8) x 10,000 requests, 2 LP + 1 HP
    cfg, b = P.workload("config2")
    assert b.T == 8 and b.R == 80_000
    assert_parity(oracle, cfg, b, gpu_sim(asc, cfg, b))


def test_config4_prefix_50k(asc, oracle):
    # BASELINE config 4's oracle scope: the first 50,000 requests of the
    # LongBench-shaped 1M-request trace at ~2x saturation, deep queues throughout
    cfg, b = P.workload("config4", n=50_000)
    got = gpu_sim(asc, cfg, b)
    assert int(got["evaluations"][0]) > 10 * int(got["decisions"][0])
    assert_parity(oracle, cfg, b, got)


@pytest.mark.slow
def test_config4_prefix_200k(asc, oracle):
    # a longer deep-queue prefix of config 4 (200,000 requests; the LP and HP
    # queues grow to ~6,000 entries; the oracle re-sorts them at every formation, ~90 s)
    cfg, b = P.workload("config4", n=200_000)
    got = gpu_sim(asc, cfg, b)
    assert int(got["evaluations"][0]) > 1000 * int(got["decisions"][0])
    assert_parity(oracle, cfg, b, got)


def test_config3_subgrid(asc, oracle):
    cfg, b = P.workload("config3", n=600)
    sub = b.subset(range(0, 4096, 16))          # every 16th grid point: all QPS x SLO scales
    assert_parity(oracle, cfg, sub, gpu_sim(asc, cfg, sub))


@pytest.mark.parametrize("policy", ["EDF_LAXITY", "EDF_DEADLINE", "SJF", "LJF", "FCFS"])
@pytest.mark.parametrize("drop", [0, 1])
def test_random_batches(asc, oracle, policy, drop):
    rng = np.random.default_rng(hash((policy, drop, 1)) % 2 ** 32)
    cfg = P.config(topo=P.topology(kv_blocks_lp=700, kv_blocks_hp=500),
                   flg=P.flags(policy=policy, drop=drop))
    b = SC.random_small_batch(rng, 24, 400)
    got = gpu_sim(asc, cfg, b)
    SC.check_invariants(b, got, cfg)
    assert_parity(oracle, cfg, b, got)


@pytest.mark.parametrize("variant", ["delay", "no_tickets", "no_elastic", "three_hp", "lp_only",
                                     "margin", "tiny_kv"])
def test_flag_variants(asc, oracle, variant):
    rng = np.random.default_rng(11)
    topo = dict(kv_blocks_lp=900, kv_blocks_hp=600)
    flg = {}
    if variant == "delay":
        flg = dict(offload_delay_us=30_000)
    elif variant == "no_tickets":
        flg = dict(tickets=0)
    elif variant == "no_elastic":
        flg = dict(elastic=0)
    elif variant == "three_hp":
        topo.update(n_lp=3, n_hp=3)
    elif variant == "lp_only":
        topo.update(n_hp=0)
    elif variant == "margin":
        flg = dict(offload_margin_us=400_000)
    elif variant == "tiny_kv":
        topo.update(kv_blocks_lp=420, kv_blocks_hp=400, lp_max_batch=16)
    cfg = P.config(topo=P.topology(**topo), flg=P.flags(**flg))
    b = SC.random_small_batch(rng, 16, 500)
    assert_parity(oracle, cfg, b, gpu_sim(asc, cfg, b))


def test_per_request_slo_and_host_path(asc, oracle):
    rng = np.random.default_rng(12)
    cfg = P.config(flg=P.flags(policy="EDF_DEADLINE"))
    b = SC.random_small_batch(rng, 6, 300)
    rt = rng.integers(100_000, 3_000_000, size=b.R).astype(np.int64)
    assert_parity(oracle, cfg, b, gpu_sim(asc, cfg, b, rt=rt), rt=rt)
    assert_parity(oracle, cfg, b, gpu_sim(asc, cfg, b, host=True))


def test_longbench_prefix(asc, oracle):
    # config 4 (QPS 12, ~2x saturation): queues grow past 32 entries -> deep-queue selection
    cfg, b = P.workload("config4", n=3000)
    got = gpu_sim(asc, cfg, b)
    assert int(got["evaluations"][0]) > 10 * int(got["decisions"][0])  # deep queues exercised
    assert_parity(oracle, cfg, b, got)


@pytest.mark.parametrize("policy", ["EDF_LAXITY", "SJF", "FCFS", "LJF", "EDF_DEADLINE"])
def test_overloaded_deep_queues(asc, oracle, policy):
    # heavy overload (QPS 48 on LongBench lengths, drops on/off): queues of hundreds of entries
    for drop in (0, 1):
        cfg, _ = P.workload("config4", n=10)
        cfg["flags"] = P.flags(policy=policy, drop=drop)
        b = TR.grid_batch([(7, 384, 16, 16), (8, 384, 8, 16)], 1500, "longbench", 2_500_000, 150_000)
        assert_parity(oracle, cfg, b, gpu_sim(asc, cfg, b))


def test_config3_full_scale_sampled(asc, oracle):
    """BASELINE config 3 at full size in bench.py's launch configuration; the oracle checks a
    stratified sample of traces (every 256th grid point) one by one."""
    cfg, b = P.workload("config3")
    got = gpu_sim(asc, cfg, b)
    idx = list(range(0, 4096, 256))
    sub = b.subset(idx)
    exp = oracle.simulate_batch(cfg, sub)
    for j, t in enumerate(idx):
        lo, hi = int(b.trace_off[t]), int(b.trace_off[t + 1])
        slo, shi = int(sub.trace_off[j]), int(sub.trace_off[j + 1])
        for k in ("first_token_us", "done_us", "prefill_start_us", "status"):
            assert np.array_equal(got[k][lo:hi], exp[k][slo:shi]), (t, k)
        assert got["digest"][t] == exp["digest"][j] and got["decisions"][t] == exp["decisions"][j]
    # properties that hold at any size, on every trace
    SC.check_invariants(b, got, cfg)
    assert np.all(got["total"] == 10_000)


def test_errors(asc):
    cfg, b = P.workload("config1", n=10)
    b.prompt_len[3] = 9000
    with pytest.raises(asc.AscError) as e:
        gpu_sim(asc, cfg, b)
    assert e.value.code == 2
    cfg, b = P.workload("config1", n=10)
    b.arrival_us[5] = 0
    with pytest.raises(asc.AscError) as e:
        gpu_sim(asc, cfg, b)
    assert e.value.code == 1
    empty = TR.make_batch([(np.zeros(0), np.zeros(0), np.zeros(0))], [1], [1])
    with pytest.raises(asc.AscError) as e:
        gpu_sim(asc, cfg, empty)
    assert e.value.code == 5
