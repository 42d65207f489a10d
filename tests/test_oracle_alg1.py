"""Pins for the oracle's Algorithm 1 and stateless LP step.

- SPEC S:318 worked example (break, not skip).
- An independent characterisation: with costs >= 1 the selected set is the longest prefix of
  the value order whose inclusive prefix sums stay strictly below every budget (G21).
- Hand-worked W1 (tests/golden/w1_lp_formation.json) for every policy.
- Offload boundary cases S:338-340 and the drop rule (G34).
"""
import itertools

import numpy as np
import pytest

import helpers as H

INF = (1 << 63) - 1


def test_spec_break_not_skip(oracle):
    # vals 3/2/1, tokens 50/500/10, N=100 -> only the first (the third fits but is not taken)
    sel = oracle.algorithm1([3, 2, 1], [0, 1, 2], [1, 1, 1], [1, 1, 1], [50, 500, 10],
                            INF, 10 ** 6, 100, 10)
    assert sel == [0]


def test_empty_and_zero_budgets(oracle):
    assert oracle.algorithm1([], [], [], [], [], INF, 10, 10, 10) == []
    assert oracle.algorithm1([1, 2], [0, 1], [1, 1], [1, 1], [1, 1], 0, 0, 0, 5) == []
    assert oracle.algorithm1([1, 2], [0, 1], [1, 1], [1, 1], [1, 1], INF, 10, 10, 0) == []


def prefix_form(val, ids, c, mem, tok, C, M, N, R):
    order = sorted(range(len(val)), key=lambda i: (-val[i], ids[i]))
    k, sc, sm, sn = 0, 0, 0, 0
    for j, i in enumerate(order):
        sc += c[i]; sm += mem[i]; sn += tok[i]
        if sc < C and sm < M and sn < N and j < R:
            k = j + 1
        else:
            break
    return order[:k]


def test_alg1_equals_prefix_sum_form(oracle):
    rng = np.random.default_rng(11)
    for _ in range(10_000):
        n = int(rng.integers(0, 9))
        val = [int(x) for x in rng.integers(-5, 5, size=n)]          # many ties
        ids = list(range(n))
        c = [int(x) for x in rng.integers(1, 20, size=n)]
        mem = [int(x) for x in rng.integers(1, 5, size=n)]
        tok = [int(x) for x in rng.integers(1, 30, size=n)]
        C = INF if rng.random() < 0.3 else int(rng.integers(0, 60))
        M, N, R = (int(rng.integers(0, 15)), int(rng.integers(0, 80)), int(rng.integers(0, 9)))
        got = oracle.algorithm1(val, ids, c, mem, tok, C, M, N, R)
        assert got == prefix_form(val, ids, c, mem, tok, C, M, N, R)
        # budget safety: strict sums below each budget, count <= R
        assert sum(tok[i] for i in got) < max(N, 1) or not got
        assert sum(mem[i] for i in got) < max(M, 1) or not got
        assert len(got) <= R
        # value-order prefix property: no skipped higher-priority request
        order = sorted(range(n), key=lambda i: (-val[i], ids[i]))
        assert got == order[:len(got)]


@pytest.mark.parametrize("policy", ["EDF_LAXITY", "EDF_DEADLINE", "FCFS", "SJF", "LJF"])
def test_w1_hand_worked(oracle, policy):
    cfg, ins, exp, rid = H.w1_step_inputs(policy)
    out = oracle.schedule_step(cfg, **ins)
    adm, off, drp = H.segment_lists(out, ins["seg_off"])[0]
    assert [rid[i] for i in adm] == exp["admitted"]
    assert [rid[i] for i in off] == exp["offloaded"]
    assert drp == []
    assert out["batch_lat_us"][0] == exp["batch_lat"] * H.SEC
    # prefill_us = 6 + 15 p (TINY-LINEAR)
    assert list(out["prefill_us"]) == [(6 + 15 * int(p)) * H.SEC for p in ins["eff_prompt"]]


def _one(oracle, cfg, dl, eff, flags, now=0):
    n = len(dl)
    return oracle.schedule_step(cfg, seg_off=[0, n], now_us=[now], deadline_us=dl,
                                eff_prompt=eff, flags=flags, dec_count=[0], dec_ctx_sum=[0],
                                tbt_slo_us=[0], budget_tokens=[0], budget_blocks=[0],
                                budget_reqs=[0])


def test_offload_boundaries(oracle):
    # S:338-340.  Zero budgets -> nothing admitted; W_hp = 6 + 15*4 = 66 s; prefill(1) = 21 s.
    big = H.tiny_cfg(margin=10 ** 15)
    r = _one(oracle, big, [10 ** 12] * 3, [1, 1, 1], [0, 0, 0])
    assert list(r["offload_idx"][:r["offload_cnt"][0]]) == [0, 1, 2]
    r = _one(oracle, H.tiny_cfg(), [100 * H.SEC + 87 * H.SEC], [1], [0])   # slack 187 s
    assert r["offload_cnt"][0] == 0
    r = _one(oracle, H.tiny_cfg(), [87 * H.SEC], [1], [0])                  # slack == 21 + 66
    assert r["offload_cnt"][0] == 1
    r = _one(oracle, H.tiny_cfg(), [87 * H.SEC + 1], [1], [0])
    assert r["offload_cnt"][0] == 0
    # ineligible: ever prefilled (bit0) or already on HP (bit1); offload disabled; no HP
    r = _one(oracle, H.tiny_cfg(), [0, 0, 0], [1, 1, 1], [1, 2, 0])
    assert list(r["offload_idx"][:r["offload_cnt"][0]]) == [2]
    assert _one(oracle, H.tiny_cfg(offload=0), [0], [1], [0])["offload_cnt"][0] == 0
    assert _one(oracle, H.tiny_cfg(n_hp=0), [0], [1], [0])["offload_cnt"][0] == 0


def test_drop_rule(oracle):
    # P:614 / G34: strictly past the deadline, never prefilled, drop mode on
    cfg = H.tiny_cfg(drop=1, offload=0)
    r = _one(oracle, cfg, [99, 100, 101, 50], [1, 1, 1, 1], [0, 0, 0, 1], now=100)
    assert list(r["drop_idx"][:r["drop_cnt"][0]]) == [0]
    assert _one(oracle, H.tiny_cfg(drop=0), [0], [1], [0], now=100)["drop_cnt"][0] == 0


def test_dropped_never_admitted_and_admitted_never_offloaded(oracle):
    rng = np.random.default_rng(5)
    from gen import presets as P
    for pol in ("EDF_LAXITY", "SJF", "FCFS"):
        cfg = P.config(flg=P.flags(policy=pol, drop=1))
        ins = H.random_step_inputs(rng, 50, 40, cfg)
        out = oracle.schedule_step(cfg, **ins)
        for adm, off, drp in H.segment_lists(out, ins["seg_off"]):
            assert not set(adm) & set(off) and not set(adm) & set(drp) and not set(off) & set(drp)
            assert off == sorted(off) and drp == sorted(drp)


def test_brute_force_alg1_optimal_under_single_budget(oracle):
    """With only the request budget R binding and SJF keys, Algorithm 1's prefix is the set of
    the R shortest prefills: brute force over all subsets of size R picks the same cost set."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        n = int(rng.integers(1, 8))
        R = int(rng.integers(1, n + 1))
        c = [int(x) for x in rng.integers(1, 50, size=n)]
        sel = oracle.algorithm1([-x for x in c], list(range(n)), c, [1] * n, [1] * n,
                                INF, 10 ** 6, 10 ** 6, R)
        best = min(sum(c[i] for i in comb) for comb in itertools.combinations(range(n), R))
        assert len(sel) == R and sum(c[i] for i in sel) == best
