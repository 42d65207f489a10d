"""SURVEY §8(d) config-4 self-check at full scale: formations sampled from the simulator's
incremental sorted-queue path (asc_simulate_batch) are replayed through the stateless decision
(asc_schedule_step: every queued request re-evaluated, selected and admitted from scratch) and
through the CPU oracle's stateless step; admitted ids (priority order), offloaded ids and the batch
latency must be identical.  asc_arm_snapshots records each sampled formation's queue and budgets."""
import numpy as np
import pytest

from gen import presets as P

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def asc():
    from paper_2504_20828_b200 import asc as A
    assert torch.cuda.is_available()
    return A


def replay(asc, oracle, cfg, snap):
    ns = int(snap["counts"][0].item())
    hdr = snap["hdr"][:16 * ns].view(ns, 16).cpu().numpy()
    ids = snap["ids"].cpu().numpy()
    dl = snap["deadline_us"].cpu().numpy()
    eff = snap["eff_prompt"].cpu().numpy()
    fl = snap["flags"].cpu().numpy()
    out_ids = snap["out_ids"].cpu().numpy()
    keep = [s for s in range(ns) if hdr[s, 10] >= 0]
    segs, order = [], []
    for s in keep:
        e0, q = int(hdr[s, 9]), int(hdr[s, 8])
        o = e0 + np.argsort(ids[e0:e0 + q], kind="stable")  # positions = ascending request id
        order.append(o)
        segs.append(q)
    off = np.zeros(len(keep) + 1, np.int64)
    off[1:] = np.cumsum(segs)
    allo = np.concatenate(order) if order else np.zeros(0, np.int64)
    h = hdr[keep]
    ins = dict(seg_off=off, now_us=h[:, 0].copy(), deadline_us=dl[allo], eff_prompt=eff[allo],
               flags=fl[allo], dec_count=h[:, 4].astype(np.int32), dec_ctx_sum=h[:, 5].copy(),
               tbt_slo_us=h[:, 6].copy(), budget_tokens=h[:, 2].astype(np.int32),
               budget_blocks=h[:, 3].astype(np.int32), budget_reqs=h[:, 7].astype(np.int32))
    ctx = asc.Context(cfg, 0)
    try:
        got = ctx.schedule_step({k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in ins.items()})
        got = {k: (v.cpu().numpy() if v is not None else None) for k, v in got.items()}
    finally:
        ctx.close()
    exp = oracle.schedule_step(cfg, **ins)
    sid = ids[allo]
    for j, s in enumerate(keep):
        lo = int(off[j])
        nadm, noff, o0 = int(hdr[s, 10]), int(hdr[s, 11]), int(hdr[s, 12])
        sim_adm = list(out_ids[o0:o0 + nadm])
        sim_off = list(out_ids[o0 + nadm:o0 + nadm + noff])
        for res, who in ((got, "asc_schedule_step"), (exp, "oracle")):
            a = res["admit_idx"][lo:lo + int(res["admit_cnt"][j])]
            f = res["offload_idx"][lo:lo + int(res["offload_cnt"][j])]
            assert list(sid[a]) == sim_adm, (who, "admitted", s, int(hdr[s, 14]))
            assert list(sid[f]) == sim_off, (who, "offloaded", s, int(hdr[s, 14]))
            assert int(res["batch_lat_us"][j]) == int(hdr[s, 13]), (who, "latency", s)
    return len(keep), int(h[:, 8].max()) if len(keep) else 0


def test_snapshot_replay_config4_prefix(asc, oracle):
    cfg, b = P.workload("config4", n=200_000)
    ctx = asc.Context(cfg, 0)
    tr = asc.batch_arrays(b, "cuda:0")
    snap = ctx.arm_snapshots(0, 0, 30011, 64, 4_000_000, 1_000_000)
    ctx.simulate_batch(tr)
    torch.cuda.synchronize()
    ctx.close()
    n, qmax = replay(asc, oracle, cfg, snap)
    assert n >= 10 and qmax >= 8, (n, qmax)


@pytest.mark.slow
def test_snapshot_replay_config4_full_scale(asc, oracle):
    """Config 4 in full (10^6 LongBench-shaped requests, QPS 12): about 20 Algorithm-1 formations of
    LP instance 0 spread over the whole run, each replayed statelessly.  (Under this load the deep
    queue is the HP instance's FCFS queue of offloaded requests; the LP queues stay short because
    urgent requests leave them.)"""
    cfg, b = P.workload("config4")
    ctx = asc.Context(cfg, 0)
    tr = asc.batch_arrays(b, "cuda:0")
    snap = ctx.arm_snapshots(0, 0, 1 << 18, 40, 8_000_000, 4_000_000)
    ctx.simulate_batch(tr)
    torch.cuda.synchronize()
    ctx.close()
    n, qmax = replay(asc, oracle, cfg, snap)
    assert n >= 10 and qmax >= 8, (n, qmax)
