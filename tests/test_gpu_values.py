"""GPU parity of row f4 (DESIGN G50-G51): weighted value functions, per-request class offsets and
the look-ahead offload rule, under Ascendra and the baselines."""
import numpy as np
import pytest

import simcases as SC
from gen import presets as P
from test_gpu_sim import gpu_sim

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def asc():
    from paper_2504_20828_b200 import asc as A
    assert torch.cuda.is_available()
    return A


def sim_off(asc, cfg, b, koff=None):
    ctx = asc.Context(cfg, 0)
    try:
        tr = asc.batch_arrays(b, "cuda:0")
        d = None if koff is None else torch.from_numpy(koff).cuda()
        out = ctx.simulate_batch(tr, req_key_offset_us=d)
        out = {k: v.cpu().numpy() for k, v in out.items()}
    finally:
        ctx.close()
    R, T = b.R, b.T
    res = {k: out[k][:R] for k in ("first_token_us", "done_us", "prefill_start_us")}
    res["status"] = out["status"][:R].view(np.uint32)
    res["digest"] = out["digest"][:T].view(np.uint64)
    res["decisions"] = out["decisions"][:T]
    res["evaluations"] = out["evaluations"][:T]
    return res


def _parity(oracle, cfg, b, got, koff=None):
    exp = oracle.simulate_batch(cfg, b, req_key_offset_us=koff)
    for k in ("first_token_us", "done_us", "prefill_start_us", "status", "digest", "decisions",
              "evaluations"):
        assert np.array_equal(got[k], exp[k]), k


def test_w8_gpu(asc):
    SC.check_w8(lambda cfg, b, rt=None: gpu_sim(asc, cfg, b, rt), lambda b, o: (o["good"], o["total"]))


@pytest.mark.parametrize("w", [(1, -1, 0), (2, -3, 0), (0, 1, 1), (1, 1, -1), (0, 0, 0), (-1, 0, 2)])
@pytest.mark.parametrize("rule", [0, 1])
def test_weighted_and_lookahead_parity(asc, oracle, w, rule):
    rng = np.random.default_rng(hash((w, rule, 51)) % 2 ** 32)
    cfg = P.config(topo=P.topology(kv_blocks_lp=700, kv_blocks_hp=500),
                   flg=P.flags(policy="WEIGHTED", key_weights=w, offload_rule=rule, drop=rule))
    b = SC.random_small_batch(rng, 20, 400)
    got = sim_off(asc, cfg, b)
    SC.check_invariants(b, got, cfg)
    _parity(oracle, cfg, b, got)


@pytest.mark.parametrize("policy", ["EDF_LAXITY", "SJF", "FCFS"])
@pytest.mark.parametrize("scheduler", ["ascendra", "vllm", "sarathi"])
def test_class_offsets_parity(asc, oracle, policy, scheduler):
    rng = np.random.default_rng(hash((policy, scheduler, 52)) % 2 ** 32)
    cfg = P.config(topo=P.topology(kv_blocks_lp=700, kv_blocks_hp=500), flg=P.flags(policy=policy))
    if scheduler != "ascendra":
        cfg = SC.with_scheduler(cfg, scheduler)
    b = SC.random_small_batch(rng, 16, 400)
    koff = SC.class_offsets(b, 5)
    _parity(oracle, cfg, b, sim_off(asc, cfg, b, koff), koff)


def test_lookahead_longbench_prefix(asc, oracle):
    cfg, b = P.workload("config4", n=3000)
    cfg["flags"] = P.flags(offload_rule=1)
    koff = SC.class_offsets(b, 7)
    _parity(oracle, cfg, b, sim_off(asc, cfg, b, koff), koff)
