"""GPU parity of the baseline schedulers in asc_simulate_batch (DESIGN G46).

Same bar as the Ascendra path: per-request times, status words, digests, decision and
evaluation counts equal the oracle's bit for bit; the hand-stepped W6 trace and the textbook
reductions pin the GPU path directly.
"""
import numpy as np
import pytest

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


def test_w6_gpu(asc):
    SC.check_fixture(lambda cfg, b, rt=None: gpu_sim(asc, cfg, b, rt),
                     lambda b, o: (o["good"], o["total"]), "w6_vllm_decode_stall.json")


def test_vllm_reductions_gpu(asc):
    rng = np.random.default_rng(5)
    for n in (1, 40, 200):
        cfg, b, end = SC.lindley_case(rng, n)
        got = gpu_sim(asc, SC.with_scheduler(cfg, "vllm"), b)
        assert [int(x) for x in got["first_token_us"]] == end
    for p, o in [(1, 1), (17, 40), (300, 7)]:
        cfg, b, first, done = SC.single_request_case(p, o)
        r = gpu_sim(asc, SC.with_scheduler(cfg, "vllm"), b)
        assert int(r["first_token_us"][0]) == first and int(r["done_us"][0]) == done


def test_vllm_fcfs_order_gpu(asc):
    SC.check_vllm_fcfs_order(lambda cfg, b, rt=None: gpu_sim(asc, cfg, b, rt),
                             np.random.default_rng(6))


@pytest.mark.parametrize("policy", ["FCFS", "EDF_LAXITY", "SJF", "LJF", "EDF_DEADLINE"])
@pytest.mark.parametrize("drop", [0, 1])
def test_vllm_random_batches(asc, oracle, policy, drop):
    rng = np.random.default_rng(hash((policy, drop, 46)) % 2 ** 32)
    cfg = SC.with_scheduler(P.config(topo=P.topology(n_lp=3, kv_blocks_lp=700),
                                     flg=P.flags(policy=policy, drop=drop)), "vllm")
    b = SC.random_small_batch(rng, 24, 400)
    got = gpu_sim(asc, cfg, b)
    SC.check_invariants(b, got, cfg)
    assert_parity(oracle, cfg, b, got)


@pytest.mark.parametrize("variant", ["tiny_kv", "cap16", "one_instance"])
def test_vllm_pressure_variants(asc, oracle, variant):
    rng = np.random.default_rng(47)
    topo = dict(n_lp=3, kv_blocks_lp=900)
    if variant == "tiny_kv":
        topo.update(kv_blocks_lp=420)
    elif variant == "cap16":
        topo.update(lp_max_batch=16)
    else:
        topo.update(n_lp=1)
    cfg = SC.with_scheduler(P.config(topo=P.topology(**topo), flg=P.flags(policy="FCFS")), "vllm")
    b = SC.random_small_batch(rng, 16, 500)
    assert_parity(oracle, cfg, b, gpu_sim(asc, cfg, b))


def test_vllm_config3_subgrid(asc, oracle):
    cfg, b = P.workload("config3", n=600)
    cfg = SC.with_scheduler(cfg, "vllm")
    cfg["topo"]["n_lp"] = 3  # the paper's three homogeneous instances
    sub = b.subset(range(0, 4096, 16))
    assert_parity(oracle, cfg, sub, gpu_sim(asc, cfg, sub))


def test_vllm_longbench_prefix(asc, oracle):
    cfg, b = P.workload("config4", n=3000)
    cfg = SC.with_scheduler(cfg, "vllm")
    cfg["topo"]["n_lp"] = 3
    assert_parity(oracle, cfg, b, gpu_sim(asc, cfg, b))


def test_vllm_config_errors(asc):
    cfg, b = P.workload("config1", n=10)
    bad = {k: dict(v) for k, v in cfg.items()}
    bad["flags"]["scheduler"] = 1  # n_hp = 1
    with pytest.raises(asc.AscError) as e:
        asc.Context(bad, 0)
    assert e.value.code == 2


# --------------------------------------------------------------- Sarathi-like (G47, G48) ------
def test_w7_gpu(asc):
    SC.check_fixture(lambda cfg, b, rt=None: gpu_sim(asc, cfg, b, rt),
                     lambda b, o: (o["good"], o["total"]), "w7_sarathi_chunks.json")


def test_sarathi_reductions_gpu(asc):
    rng = np.random.default_rng(11)
    for n in (1, 40):
        cfg, b, end = SC.lindley_case(rng, n)
        cfg = SC.with_scheduler(cfg, "sarathi")
        cfg["flags"]["chunk_tokens"] = 64
        got = gpu_sim(asc, cfg, b)
        assert [int(x) for x in got["first_token_us"]] == end


@pytest.mark.parametrize("policy", ["FCFS", "EDF_LAXITY", "SJF", "LJF", "EDF_DEADLINE"])
@pytest.mark.parametrize("chunk", [64, 512, 2048])
def test_sarathi_random_batches(asc, oracle, policy, chunk):
    rng = np.random.default_rng(hash((policy, chunk, 47)) % 2 ** 32)
    cfg = SC.with_scheduler(P.config(topo=P.topology(n_lp=3, kv_blocks_lp=700),
                                     flg=P.flags(policy=policy, drop=int(chunk == 64),
                                                 chunk_tokens=chunk)), "sarathi")
    b = SC.random_small_batch(rng, 24, 400)
    got = gpu_sim(asc, cfg, b)
    SC.check_invariants(b, got, cfg)
    assert_parity(oracle, cfg, b, got)


@pytest.mark.parametrize("variant", ["tiny_kv", "cap16", "one_instance", "chunk1"])
def test_sarathi_pressure_variants(asc, oracle, variant):
    rng = np.random.default_rng(48)
    topo = dict(n_lp=3, kv_blocks_lp=900)
    chunk = 256
    if variant == "tiny_kv":
        topo.update(kv_blocks_lp=420)
    elif variant == "cap16":
        topo.update(lp_max_batch=16)
    elif variant == "one_instance":
        topo.update(n_lp=1)
    else:
        chunk = 1  # budget below the decode count: prefill waits for decodes to drain
    cfg = SC.with_scheduler(P.config(topo=P.topology(**topo),
                                     flg=P.flags(policy="FCFS", chunk_tokens=chunk)), "sarathi")
    b = SC.random_small_batch(rng, 16, 300 if variant == "chunk1" else 500)
    assert_parity(oracle, cfg, b, gpu_sim(asc, cfg, b))


def test_sarathi_config3_subgrid(asc, oracle):
    cfg, b = P.workload("config3", n=600)
    cfg = SC.with_scheduler(cfg, "sarathi")
    cfg["topo"]["n_lp"] = 3
    sub = b.subset(range(0, 4096, 16))
    assert_parity(oracle, cfg, sub, gpu_sim(asc, cfg, sub))


def test_sarathi_longbench_prefix(asc, oracle):
    cfg, b = P.workload("config4", n=3000)
    cfg = SC.with_scheduler(cfg, "sarathi")
    cfg["topo"]["n_lp"] = 3
    cfg["flags"]["chunk_tokens"] = 2048
    assert_parity(oracle, cfg, b, gpu_sim(asc, cfg, b))


@pytest.mark.parametrize("sched", ["vllm", "sarathi"])
def test_baselines_config2_full(asc, oracle, sched):
    # BASELINE config 2 at full size (8 traces, QPS 1..8, 10k requests each) on the paper's three
    # homogeneous instances, both baseline schedulers
    cfg, b = P.workload("config2")
    cfg = SC.with_scheduler(cfg, sched)
    cfg["topo"]["n_lp"] = 3
    assert_parity(oracle, cfg, b, gpu_sim(asc, cfg, b))
