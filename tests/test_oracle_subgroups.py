"""Per-trace subgroup topology (row f3; "scale the system using subgroups",
Fig scale_fig: 1L1H, 2L1H, 1L2H).  A batch mixing topologies must give every trace exactly what
a run of that trace alone, under its topology, gives; the Lindley reduction holds per trace."""
import numpy as np
import pytest

import simcases as SC
from gen import presets as P
from gen import traces as TR

TOPOS = [(1, 0), (1, 1), (2, 1), (1, 2), (3, 0), (2, 0)]


def topo_arrays(T, rng):
    pick = rng.integers(0, len(TOPOS), size=T)
    return (np.array([TOPOS[i][0] for i in pick], np.int32), np.array([TOPOS[i][1] for i in pick], np.int32))


def test_mixed_topologies_equal_separate_runs(oracle):
    rng = np.random.default_rng(30)
    cfg = P.config(topo=P.topology(n_lp=2, n_hp=1, kv_blocks_lp=900, kv_blocks_hp=700))
    b = SC.random_small_batch(rng, 12, 300)
    nl, nh = topo_arrays(b.T, rng)
    out = oracle.simulate_batch(cfg, b, n_lp=nl, n_hp=nh, check_invariants=True)
    for t in range(b.T):
        c = {k: dict(v) for k, v in cfg.items()}
        c["topo"].update(n_lp=int(nl[t]), n_hp=int(nh[t]))
        one = b.subset([t])
        exp = oracle.simulate_batch(c, one)
        lo, hi = int(b.trace_off[t]), int(b.trace_off[t + 1])
        for k in ("first_token_us", "done_us", "prefill_start_us", "status"):
            assert np.array_equal(out[k][lo:hi], exp[k]), (t, k)
        for k in ("digest", "decisions", "evaluations"):
            assert out[k][t] == exp[k][0], (t, k)


def test_lindley_trace_inside_a_mixed_batch(oracle):
    rng = np.random.default_rng(31)
    cfg, bl, end = SC.lindley_case(rng, 50)  # 1 LP, no HP, cap 1, output 1
    cfg = {k: dict(v) for k, v in cfg.items()}
    cfg["topo"].update(n_lp=2, n_hp=1)       # the pool; the Lindley trace uses 1L0H
    trs = [bl.trace(0)[:3]]
    for _ in range(2):  # small prompts: the TINY config's token budget is 64
        n = 40
        arr = np.sort(rng.integers(0, 10 ** 8, size=n)).astype(np.int64)
        trs.append((arr, rng.integers(1, 30, size=n), rng.integers(1, 20, size=n)))
    b = TR.make_batch(trs, [int(bl.ttft_slo_us[0])] * 3, [int(bl.tbt_slo_us[0])] * 3)
    out = oracle.simulate_batch(cfg, b, n_lp=np.array([1, 2, 1], np.int32),
                                n_hp=np.array([0, 1, 2], np.int32))
    assert [int(x) for x in out["first_token_us"][:50]] == end


@pytest.mark.parametrize("nl,nh", [(0, 1), (3, 1), (2, -1)])
def test_topology_out_of_range(oracle, nl, nh):
    cfg, b = P.workload("config1", n=10)  # pool 1L1H
    with pytest.raises(oracle.OracleError):
        oracle.simulate_batch(cfg, b, n_lp=np.array([nl], np.int32), n_hp=np.array([nh], np.int32))
