"""Row e on one GPU: the config-5 grid sharded i = rank (mod W) as bench.py shards it under
torchrun.  Each shard is its own asc_simulate_batch call (one per "rank"); reassembled per-trace
digests, decisions, outcomes and goodput counters must equal the unsharded call's for W = 2, 4, 8
and the oracle's on the same traces ("cross-GPU-count digest equality")."""
import numpy as np
import pytest

from gen import presets as P
from paper_2504_20828_b200 import dist as D

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _run(asc, cfg, b):
    ctx = asc.Context(cfg, 0)
    try:
        tr = asc.batch_arrays(b, "cuda:0")
        out = ctx.simulate_batch(tr)
        good, total = ctx.goodput(tr, out)
        res = {k: v.cpu().numpy() for k, v in out.items()}
        res["good"], res["total"] = good.cpu().numpy(), total.cpu().numpy()
    finally:
        ctx.close()
    T, R = b.T, b.R
    return {"digest": res["digest"][:T].view(np.uint64), "decisions": res["decisions"][:T],
            "good": res["good"][:T].view(np.uint64), "total": res["total"][:T].view(np.uint64),
            "first_token_us": res["first_token_us"][:R], "done_us": res["done_us"][:R],
            "status": res["status"][:R].view(np.uint32)}


def test_config5_shards_match_unsharded_and_oracle():
    from paper_2504_20828_b200 import asc
    from oracle import oracle as O
    # every 64th grid point of the 65,536-trace config-5 grid (all QPS values, all SLO scales)
    cfg, full = P.workload("config5", n=1)
    idx = list(range(0, full.T, 64))
    cfg, b5 = P.workload("config5", n=400)
    b = b5.subset(idx)
    whole = _run(asc, cfg, b)
    exp = O.simulate_batch(cfg, b)
    assert np.array_equal(whole["digest"], exp["digest"])
    assert np.array_equal(whole["decisions"], exp["decisions"])
    assert np.array_equal(whole["first_token_us"], exp["first_token_us"])
    assert np.array_equal(whole["done_us"], exp["done_us"])
    assert np.array_equal(whole["status"], exp["status"])
    off = np.asarray(b.trace_off)
    for W in (2, 4, 8):
        dig = np.zeros(b.T, np.uint64)
        dec = np.zeros(b.T, np.int64)
        first = np.full(b.R, -2, np.int64)
        sums = {"good": 0, "total": 0}
        for r in range(W):
            sh = D.shard(b.T, r, W)
            got = _run(asc, cfg, b.subset(sh))
            dig[sh] = got["digest"]
            dec[sh] = got["decisions"]
            pos = 0
            for t in sh:  # the shard's requests, in its trace order
                n = int(off[t + 1] - off[t])
                first[off[t]:off[t + 1]] = got["first_token_us"][pos:pos + n]
                pos += n
            sums["good"] += int(got["good"].sum())
            sums["total"] += int(got["total"].sum())
        assert np.array_equal(dig, whole["digest"]), W
        assert np.array_equal(dec, whole["decisions"]), W
        assert np.array_equal(first, whole["first_token_us"]), W
        assert sums["good"] == int(whole["good"].sum()) and sums["total"] == int(whole["total"].sum())


def test_more_traces_than_resident_warps():
    """8,192 traces (the per-GPU load of config 5 on 8 GPUs) exceed the resident warp slots
    (148 SMs x 7 CTAs x 4 warps): warps pull further traces from the atomic counter."""
    from paper_2504_20828_b200 import asc
    from oracle import oracle as O
    cfg, b = P.workload("config5", n=60, select=list(range(0, 65536, 8)))
    assert b.T == 8192
    got = _run(asc, cfg, b)
    exp = O.simulate_batch(cfg, b)
    assert np.array_equal(got["digest"], exp["digest"])
    assert np.array_equal(got["decisions"], exp["decisions"])
    assert np.array_equal(got["first_token_us"], exp["first_token_us"])
    assert np.array_equal(got["done_us"], exp["done_us"])
    assert np.array_equal(got["status"], exp["status"])
