"""GPU parity of per-trace subgroup topology in asc_simulate_batch (row f3)."""
import numpy as np
import pytest

import simcases as SC
from gen import presets as P
from test_gpu_sim import assert_parity
from test_oracle_subgroups import topo_arrays

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def asc():
    from paper_2504_20828_b200 import asc as A
    assert torch.cuda.is_available()
    return A


def sim_topo(asc, cfg, b, nl, nh, host=False):
    ctx = asc.Context(cfg, 0)
    try:
        if host:
            tr = asc.batch_arrays(b)
            out = ctx.simulate_batch(tr, n_lp=nl, n_hp=nh)
            good, total = ctx.goodput(tr, out)
        else:
            tr = asc.batch_arrays(b, "cuda:0")
            dn = lambda a: torch.from_numpy(a).cuda()
            out = ctx.simulate_batch(tr, n_lp=dn(nl), n_hp=dn(nh))
            good, total = ctx.goodput(tr, out)
            out = {k: v.cpu().numpy() for k, v in out.items()}
            good, total = good.cpu().numpy(), total.cpu().numpy()
    finally:
        ctx.close()
    R, T = b.R, b.T
    res = {k: out[k][:R] for k in ("first_token_us", "done_us", "prefill_start_us")}
    res["status"] = out["status"][:R].view(np.uint32)
    res["digest"] = out["digest"][:T].view(np.uint64)
    res["decisions"] = out["decisions"][:T]
    res["evaluations"] = out["evaluations"][:T]
    res["good"] = good[:T].view(np.uint64)
    res["total"] = total[:T].view(np.uint64)
    return res


def _parity(oracle, cfg, b, nl, nh, got):
    exp = oracle.simulate_batch(cfg, b, n_lp=nl, n_hp=nh)
    for k in ("first_token_us", "done_us", "prefill_start_us", "status", "digest", "decisions",
              "evaluations"):
        assert np.array_equal(got[k], exp[k]), k


@pytest.mark.parametrize("policy", ["EDF_LAXITY", "SJF", "FCFS"])
def test_mixed_topologies_gpu(asc, oracle, policy):
    rng = np.random.default_rng(hash((policy, 32)) % 2 ** 32)
    cfg = P.config(topo=P.topology(n_lp=2, n_hp=1, kv_blocks_lp=800, kv_blocks_hp=600),
                   flg=P.flags(policy=policy))
    b = SC.random_small_batch(rng, 30, 400)
    nl, nh = topo_arrays(b.T, rng)
    got = sim_topo(asc, cfg, b, nl, nh)
    _parity(oracle, cfg, b, nl, nh, got)
    _parity(oracle, cfg, b, nl, nh, sim_topo(asc, cfg, b, nl, nh, host=True))


def test_config3_subgrid_topology_axis(asc, oracle):
    # config 3's grid with the subgroup topology as one more axis (pool of 3 instances)
    cfg, b = P.workload("config3", n=600)
    sub = b.subset(range(0, 4096, 16))
    T = sub.T
    topos = [(3, 0), (2, 1), (1, 2)]
    nl = np.array([topos[t % 3][0] for t in range(T)], np.int32)
    nh = np.array([topos[t % 3][1] for t in range(T)], np.int32)
    _parity(oracle, cfg, sub, nl, nh, sim_topo(asc, cfg, sub, nl, nh))


def test_topology_errors_gpu(asc):
    cfg, b = P.workload("config1", n=10)
    with pytest.raises(asc.AscError) as e:
        sim_topo(asc, cfg, b, np.array([2], np.int32), np.array([1], np.int32))
    assert e.value.code == 2
