"""Pins for the oracle's baseline schedulers (reading G46).

vLLM-like: hand-stepped decode stall (W6), the Lindley FCFS queue and the single-request closed
form (both reduce to textbook results when nothing overlaps), FCFS order preservation,
invariants under pressure, and configuration errors.
"""
import numpy as np
import pytest

import helpers as H
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


# --------------------------------------------------------------- Sarathi-like (G47, G48) ------
def test_w7_sarathi_chunks(oracle):
    SC.check_fixture(_sim(oracle), oracle.goodput, "w7_sarathi_chunks.json")


def test_chunked_cost_reduces_to_whole_prompts(oracle):
    # G48: chunks with no cached context cost exactly what Eq. 1-3 charge for whole prompts
    rng = np.random.default_rng(8)
    for arch in (P.MISTRAL7B, P.TINY):
        for _ in range(20):
            p = rng.integers(1, 4000, size=int(rng.integers(1, 6)))
            lh = rng.integers(1, 5000, size=int(rng.integers(0, 9)))
            F, M, rc = oracle.cost_chunked(arch, np.zeros(len(p)), p, lh)
            F2, M2, rc2 = oracle.cost(arch, p, lh)
            assert (F, M, rc) == (F2, M2, rc2)
        assert oracle.cost_chunked(arch, [], [], [])[:2] == oracle.cost(arch, [], [])[:2]


def test_chunk_sum_identity(oracle):
    # splitting a prompt p into chunks keeps the GEMM terms and the cached-context
    # loads; attention flops drop by exactly 2 s n L sum_j l_j c_j (l_j = tokens before chunk j),
    # since p^2 = sum c_j^2 + 2 sum_j l_j c_j.  Checked on one attention head, one layer.
    a = dict(P.MISTRAL7B, L=1, n=1, h=128, s=128, n_kv=1, m=1)
    rng = np.random.default_rng(9)
    for _ in range(30):
        p = int(rng.integers(2, 3000))
        cuts = np.sort(rng.choice(np.arange(1, p), size=min(int(rng.integers(1, 5)), p - 1), replace=False))
        c = np.diff(np.concatenate([[0], cuts, [p]]))
        l = np.concatenate([[0], np.cumsum(c)[:-1]])
        s = a["s"]
        # each chunk as its own batch (the way a request is chunked across batches)
        Fsum = sum(oracle.cost_chunked(a, [int(li)], [int(ci)])[0] for li, ci in zip(l, c))
        Fw = oracle.cost(a, [p])[0]
        gemm1 = 4 * a["h"] ** 2 + 2 * a["h"] * a["m"]  # flops per token per layer (Tables 3-4)
        attn_whole = 2 * s * p * p
        attn_chunks = sum(2 * s * (int(li) * int(ci) + int(ci) ** 2) for li, ci in zip(l, c))
        assert Fw == gemm1 * p + attn_whole
        assert Fsum == gemm1 * p + attn_chunks
        assert attn_whole - attn_chunks == 2 * s * int(np.dot(l, c))


def test_chunked_cost_tiny_closed_form(oracle):
    # TINY-LINEAR: latency seconds = M = 6 + sum_chunks (15c + 2l + 3c [l > 0]) + sum_dec (12 + 2 lhat)
    rng = np.random.default_rng(10)
    for _ in range(50):
        k = int(rng.integers(0, 4))
        l = rng.integers(0, 50, size=k)
        c = rng.integers(1, 50, size=k)
        lh = rng.integers(1, 60, size=int(rng.integers(0 if k else 1, 5)))
        _, M, _ = oracle.cost_chunked(P.TINY, l, c, lh)
        exp = 6 + sum(15 * int(ci) + 2 * int(li) + 3 * int(ci) * (li > 0) for li, ci in zip(l, c)) \
            + sum(12 + 2 * int(x) for x in lh)
        assert M == exp


def test_sarathi_whole_prompt_budget_equals_lindley(oracle):
    # a budget covering every prompt and batch cap 1, output 1: each batch is one whole prompt,
    # so Sarathi-like is the single-server FCFS queue too (Lindley recursion)
    rng = np.random.default_rng(11)
    for n in (1, 3, 40):
        cfg, b, end = SC.lindley_case(rng, n)
        cfg = SC.with_scheduler(cfg, "sarathi")
        cfg["flags"]["chunk_tokens"] = 64
        out = _sim(oracle)(cfg, b)
        assert [int(x) for x in out["first_token_us"]] == end


def test_sarathi_single_request_chunks(oracle):
    # one request of p tokens under budget B: ceil(p / B) chunk batches, then decodes; TINY
    for p, B, o in [(10, 4, 3), (7, 7, 1), (33, 5, 4), (1, 512, 2)]:
        cfg, b, _, _ = SC.single_request_case(p, o)
        cfg = SC.with_scheduler(cfg, "sarathi")
        cfg["flags"]["chunk_tokens"] = B
        out = _sim(oracle)(cfg, b)
        t, l = 7, 0
        while l < p:
            c = min(B, p - l)
            t += 6 + 15 * c + 2 * l + 3 * c * (l > 0)
            l += c
        first = t
        for g in range(1, o):
            t += 6 + 12 + 2 * (p + g)
        assert int(out["first_token_us"][0]) == first * H.SEC and int(out["done_us"][0]) == t * H.SEC


@pytest.mark.parametrize("policy", ["FCFS", "SJF", "EDF_LAXITY"])
def test_sarathi_invariants_under_pressure(oracle, policy):
    cfg = SC.with_scheduler(P.config(topo=P.topology(n_lp=3, kv_blocks_lp=450),
                                     flg=P.flags(policy=policy, drop=1, chunk_tokens=256)), "sarathi")
    _, b = P.workload("config2", n=400)
    out = _sim(oracle)(cfg, b)
    SC.check_invariants(b, out, cfg)
    assert SC.npre(out["status"]).sum() > 0
