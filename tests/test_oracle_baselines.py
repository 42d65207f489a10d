"""Pins for the oracle's baseline schedulers (reading G46).

vLLM-like: hand-stepped decode stall (W6), the Lindley FCFS queue and the single-request closed
form (both reduce to textbook results when nothing overlaps), FCFS order preservation,
invariants under pressure, and configuration errors.
"""
import numpy as np
import pytest

import simcases as SC
from gen import presets as P


def _sim(oracle):
    return lambda cfg, b, rt=None: oracle.simulate_batch(cfg, b, req_ttft_slo_us=rt,
                                                         check_invariants=True)


def test_w6_vllm_decode_stall(oracle):
    SC.check_fixture(_sim(oracle), oracle.goodput, "w6_vllm_decode_stall.json")


def test_vllm_lindley(oracle):
    rng = np.random.default_rng(5)
    for n in (1, 3, 40, 200):
        cfg, b, end = SC.lindley_case(rng, n)
        out = _sim(oracle)(SC.with_scheduler(cfg, "vllm"), b)
        assert [int(x) for x in out["first_token_us"]] == end
        assert [int(x) for x in out["done_us"]] == end


@pytest.mark.parametrize("p,o", [(1, 1), (5, 2), (17, 40), (300, 7)])
def test_vllm_single_request_closed_form(oracle, p, o):
    cfg, b, first, done = SC.single_request_case(p, o)
    out = _sim(oracle)(SC.with_scheduler(cfg, "vllm"), b)
    assert int(out["first_token_us"][0]) == first and int(out["done_us"][0]) == done
    assert int(out["decisions"][0]) == o


def test_vllm_fcfs_order(oracle):
    SC.check_vllm_fcfs_order(_sim(oracle), np.random.default_rng(6))


@pytest.mark.parametrize("policy", ["FCFS", "SJF", "EDF_LAXITY"])
def test_vllm_invariants_under_pressure(oracle, policy):
    cfg = SC.with_scheduler(P.config(topo=P.topology(n_lp=3, kv_blocks_lp=450),
                                     flg=P.flags(policy=policy, drop=1)), "vllm")
    _, b = P.workload("config2", n=400)
    out = _sim(oracle)(cfg, b)
    SC.check_invariants(b, out, cfg)
    assert SC.npre(out["status"]).sum() > 0  # preemption by recomputation exercised


def test_vllm_config_errors(oracle):
    cfg, b = P.workload("config1", n=10)
    bad = {k: dict(v) for k, v in cfg.items()}
    bad["flags"]["scheduler"] = 1  # n_hp = 1: baselines run on homogeneous instances only
    with pytest.raises(oracle.OracleError):
        oracle.simulate_batch(bad, b)
    bad["flags"]["scheduler"] = 7
    bad["topo"]["n_hp"] = 0
    with pytest.raises(oracle.OracleError):
        oracle.simulate_batch(bad, b)
