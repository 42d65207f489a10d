"""Row f4 pins (DESIGN G50-G51): the weighted value function reduces exactly to each built-in
policy; a class offset common to every request changes nothing; premium requests (earlier keys)
see lower TTFT under load; the look-ahead offload rule against the paper's on a hand-stepped
trace (W8)."""
import numpy as np
import pytest

import simcases as SC
from gen import presets as P


def _sim(oracle):
    return lambda cfg, b, rt=None: oracle.simulate_batch(cfg, b, check_invariants=True)


def test_w8_offload_rules(oracle):
    SC.check_w8(_sim(oracle), oracle.goodput)


@pytest.mark.parametrize("w,policy", SC.WEIGHTED_EQUIV)
def test_weighted_reduces_to_policy(oracle, w, policy):
    rng = np.random.default_rng(40)
    b = SC.random_small_batch(rng, 6, 300)
    base = P.config(topo=P.topology(kv_blocks_lp=700, kv_blocks_hp=500), flg=P.flags(policy=policy, drop=1))
    wcfg = P.config(topo=P.topology(kv_blocks_lp=700, kv_blocks_hp=500),
                    flg=P.flags(policy="WEIGHTED", key_weights=w, drop=1))
    a, c = oracle.simulate_batch(base, b), oracle.simulate_batch(wcfg, b)
    for k in a:
        assert np.array_equal(a[k], c[k]), k


def test_common_offset_is_neutral(oracle):
    rng = np.random.default_rng(41)
    b = SC.random_small_batch(rng, 6, 300)
    cfg = P.config(flg=P.flags(policy="EDF_DEADLINE"))
    a = oracle.simulate_batch(cfg, b)
    c = oracle.simulate_batch(cfg, b, req_key_offset_us=np.full(b.R, -123_456_789, np.int64))
    for k in a:
        assert np.array_equal(a[k], c[k]), k


def test_premium_class_gets_lower_ttft(oracle):
    cfg, b = P.workload("config4", n=1500)  # overloaded LongBench-shaped trace
    off = SC.class_offsets(b, 3)  # default flags: EDF_LAXITY, offload on
    out = oracle.simulate_batch(cfg, b, req_key_offset_us=off)
    ttft = out["first_token_us"] - b.arrival_us
    prem = off < 0
    assert ttft[prem].mean() < 0.5 * ttft[~prem].mean()


def test_simulator_only_options_rejected_by_step(oracle):
    import helpers as H
    rng = np.random.default_rng(42)
    for flg in (P.flags(policy="WEIGHTED"), P.flags(offload_rule=1)):
        cfg = P.config(flg=flg)
        ins = H.random_step_inputs(rng, 3, 10, cfg)
        with pytest.raises(oracle.OracleError):
            oracle.schedule_step(cfg, **ins)
