"""N > 1 path on CPU: two gloo ranks shard a config-5-shaped grid, run their traces (the CPU
oracle stands in for each rank's GPU, which this container lacks) and reduce the integer
counters / gather digests; the totals and per-trace digests must equal one process's."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _work(cfg, b, idx):
    from oracle import oracle as O
    sub = b.subset(idx)
    out = O.simulate_batch(cfg, sub, nthreads=1)
    g, t = O.goodput(sub, out)
    st = out["status"] & 3
    vals = dict(decisions=int(out["decisions"].sum()), evaluations=int(out["evaluations"].sum()),
                finished=int((st != 0).sum()), good=int(g.sum()), total=int(t.sum()), requests=sub.R)
    return vals, out["digest"].view(np.int64)


def _rank(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from gen import presets as P
    from paper_2504_20828_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, b = P.workload("config5", n=150, max_traces=40)
    vals, dig = _work(cfg, b, D.shard(b.T, rank, world))
    tot = D.reduce_counters(vals, "cpu")
    tmax = D.reduce_max(1.0 + rank, "cpu")
    parts = D.gather_digests(dig, "cpu")
    if rank == 0:
        q.put((tot, tmax, [p.numpy().tolist() for p in parts]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_matches_single_process():
    sys.path.insert(0, ROOT)
    from gen import presets as P
    from paper_2504_20828_b200 import dist as D
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    tot, tmax, parts = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg, b = P.workload("config5", n=150, max_traces=40)
    ref, dig = _work(cfg, b, list(range(b.T)))
    assert tot == ref
    assert tmax == 2.0
    # reassemble the interleaved shards into global trace order
    glob = np.zeros(b.T, np.int64)
    for r in range(world):
        glob[D.shard(b.T, r, world)] = parts[r]
    assert np.array_equal(glob, dig)


def _per_trace(cfg, b, idx):
    """The per-trace arrays bench.py feeds to D.point_counters (oracle stands in for the GPU)."""
    from oracle import oracle as O
    sub = b.subset(idx)
    out = O.simulate_batch(cfg, sub, nthreads=1)
    g, t = O.goodput(sub, out)
    s = O.summarize(cfg, sub, out)
    pt = dict(good=g.astype(np.int64), total=t.astype(np.int64), decisions=out["decisions"],
              evaluations=out["evaluations"], finished=s["completed"] + s["dropped"],
              **{k: s[k] for k in ("completed", "dropped", "tokens", "tbt_sum_us", "tbt_tokens",
                                   "delay_sum_lp_us", "delay_cnt_lp", "delay_sum_hp_us", "delay_cnt_hp")})
    rows = np.stack([out["digest"].view(np.int64), s["ttft_p99_us"]], 1)
    return pt, rows


def _point_of(b):
    # config-5 grid: trace index (qi*64 + si)*16 + seed -> point qi*64 + si
    return np.array([int(l.split(":")[0][1:]) // 16 for l in b.labels], np.int64)


def _rank_points(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from gen import presets as P
    from paper_2504_20828_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, b = P.workload("config5", n=120, max_traces=96)
    idx = D.shard(b.T, rank, world)
    pt, rows = _per_trace(cfg, b, idx)
    tab = D.reduce_points(D.point_counters(_point_of(b)[idx], 6, pt), "cpu")
    parts = D.gather_rows(rows, "cpu")
    if rank == 0:
        q.put((tab, parts))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_point_reduction_matches_single_process():
    # bench.py's per-grid-point reduction: [points x counters] int64 all-reduce and
    # the all-gather of per-trace (digest, p99 TTFT) rows; per-point goodput equals one process's
    sys.path.insert(0, ROOT)
    from gen import presets as P
    from paper_2504_20828_b200 import dist as D
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_points, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    tab, parts = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg, b = P.workload("config5", n=120, max_traces=96)
    pt, rows = _per_trace(cfg, b, list(range(b.T)))
    ref = D.point_counters(_point_of(b), 6, pt)
    assert tab.shape == (6, len(D.POINT_COUNTERS)) and np.array_equal(tab, ref)
    gi, ti = D.POINT_COUNTERS.index("good"), D.POINT_COUNTERS.index("total")
    assert (ref[:, ti] == 16 * 120).all()
    glob = np.zeros_like(rows)
    for r in range(world):
        glob[D.shard(b.T, r, world)] = parts[r]
    assert np.array_equal(glob, rows)
    # per-point goodput from the table equals the per-trace oracle goodput summed by point
    g_direct = np.bincount(_point_of(b), weights=pt["good"], minlength=6)
    assert np.array_equal(tab[:, gi], g_direct.astype(np.int64))


def test_shard_partition():
    from paper_2504_20828_b200 import dist as D
    for T in (1, 7, 4096):
        for w in (1, 2, 3, 8):
            got = sorted(i for r in range(w) for i in D.shard(T, r, w))
            assert got == list(range(T))
