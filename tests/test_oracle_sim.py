"""Pins for the oracle's batch-level simulator (§4-§6; DESIGN.md event rules).

Hand-stepped traces W2-W5 (tests/golden), the Lindley FCFS degenerate case, the single-request
closed form, textbook scheduling rules by brute force (SPT, common due date, Jackson), the
invariants of S:522-527 and determinism.
"""
import numpy as np
import pytest

import helpers as H
import simcases as SC
from gen import presets as P


def _sim(oracle):
    return lambda cfg, b, rt=None: oracle.simulate_batch(cfg, b, req_ttft_slo_us=rt,
                                                         check_invariants=True)


@pytest.mark.parametrize("name", ["w2_two_request_des.json", "w3_tickets_offload.json",
                                  "w4_preemption.json"])
def test_hand_stepped(oracle, name):
    SC.check_fixture(_sim(oracle), oracle.goodput, name)


def test_elastic_trigger(oracle):
    SC.check_elastic(_sim(oracle))


def test_lindley(oracle):
    rng = np.random.default_rng(1)
    for n in (1, 2, 5, 30, 200):
        cfg, b, end = SC.lindley_case(rng, n)
        out = _sim(oracle)(cfg, b)
        assert [int(x) for x in out["first_token_us"]] == end
        assert [int(x) for x in out["done_us"]] == end


@pytest.mark.parametrize("p,o", [(1, 1), (5, 2), (17, 40), (300, 7)])
def test_single_request_closed_form(oracle, p, o):
    cfg, b, first, done = SC.single_request_case(p, o)
    out = _sim(oracle)(cfg, b)
    assert int(out["first_token_us"][0]) == first and int(out["done_us"][0]) == done
    assert int(out["decisions"][0]) == o  # one prefill batch + (o-1) decode steps


def test_textbook_rules(oracle):
    SC.check_textbook_rules(_sim(oracle), oracle.goodput, np.random.default_rng(2))


def test_routing_round_robin(oracle):
    # no tickets, 2 LPs -> LP0, LP1, LP0, ...  (light load, no preemption)
    cfg = P.config(flg=P.flags(tickets=0, offload=0))
    cfg["topo"]["n_hp"] = 0
    _, b = P.workload("config1", n=60)
    out = _sim(oracle)(cfg, b)
    assert list(SC.inst(out["status"])) == [i % 2 for i in range(60)]


@pytest.mark.parametrize("seed", range(3))
def test_invariants_random(oracle, seed):
    rng = np.random.default_rng(seed)
    for drop in (0, 1):
        for pol in ("EDF_LAXITY", "SJF", "FCFS", "LJF", "EDF_DEADLINE"):
            cfg = P.config(topo=P.topology(kv_blocks_lp=600, kv_blocks_hp=400),
                           flg=P.flags(policy=pol, drop=drop))
            b = SC.random_small_batch(rng, 4, 300)
            out = _sim(oracle)(cfg, b)
            SC.check_invariants(b, out, cfg)


def test_preemption_occurs_under_pressure(oracle):
    cfg = P.config(topo=P.topology(kv_blocks_lp=450, kv_blocks_hp=450))
    _, b = P.workload("config2", n=400)
    out = _sim(oracle)(cfg, b)
    SC.check_invariants(b, out, cfg)
    assert SC.npre(out["status"]).sum() > 0


def test_determinism_and_threads(oracle):
    cfg, b = P.workload("config3", n=300, max_traces=24)
    o1 = oracle.simulate_batch(cfg, b, nthreads=1)
    o8 = oracle.simulate_batch(cfg, b, nthreads=8)
    for k in o1:
        assert np.array_equal(o1[k], o8[k]), k


def test_validation_errors(oracle):
    cfg, b = P.workload("config1", n=5)
    b.prompt_len[2] = 9000  # prompt + output > lp_token_budget
    with pytest.raises(oracle.OracleError) as e:
        oracle.simulate_batch(cfg, b)
    assert e.value.code == 2
    cfg, b = P.workload("config1", n=5)
    b.arrival_us[3] = 0
    with pytest.raises(oracle.OracleError):
        oracle.simulate_batch(cfg, b)
