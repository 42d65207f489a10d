"""Small invocations of every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck).  Each case is also checked against the oracle, so a run that the sanitizer passes is
also a correct one.  GPU box only; driven by tools/sanitize.sh."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import helpers as H  # noqa: E402
from gen import presets as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2504_20828_b200 import asc  # noqa: E402


def dev(ins):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in ins.items()}


def sim_case(name, n, **kw):
    cfg, b = P.workload(name, n=n, **kw)
    ctx = asc.Context(cfg, 0)
    tr = asc.batch_arrays(b, "cuda:0")
    out = ctx.simulate_batch(tr)
    good, total = ctx.goodput(tr, out)
    summ = ctx.summarize(tr, out)
    torch.cuda.synchronize()
    ref = O.simulate_batch(cfg, b)
    for k in ("first_token_us", "done_us"):
        assert np.array_equal(out[k].cpu().numpy(), ref[k]), (name, k)
    assert np.array_equal(out["digest"].cpu().numpy().view(np.uint64), ref["digest"]), name
    rg, rt = O.goodput(b, ref)
    assert np.array_equal(good.cpu().numpy().view(np.uint64)[:b.T], np.asarray(rg, np.uint64)), name
    del summ
    ctx.close()
    print("ok sim", name, n, b.T, "traces")


def step_case():
    # mixed segment sizes: k_small (<= 32), single-task k1, multi-task k1 + k2 merge + k3 expansion
    cfg = P.config(flg=P.flags(drop=1))
    rng = np.random.default_rng(7)
    qs = np.array([0, 1, 7, 32, 33, 200, 5000, 16384, 16385, 40000, 3, 31])
    ins = H.random_step_inputs(rng, len(qs), 0, cfg, qs=qs)
    ctx = asc.Context(cfg, 0)
    got = ctx.schedule_step(dev(ins))
    torch.cuda.synchronize()
    exp = O.schedule_step(cfg, **ins)
    S = len(qs)
    for k in ("admit_cnt", "offload_cnt", "drop_cnt", "batch_lat_us"):
        assert np.array_equal(got[k].cpu().numpy()[:S], exp[k][:S]), k
    ctx.close()
    print("ok step mixed", int(qs.sum()), "entries")


def lane_case():
    # k_lane: full 32-entry groups (n == 32 path), mixed short groups (general path), segments
    # handed back to k_small (a key outside the 2^26 us window, a prompt beyond the fast table),
    # and S > 8191 for the two-launch planner
    cfg = P.config(flg=P.flags(drop=1))
    rng = np.random.default_rng(11)
    S = 8300
    qs = rng.integers(0, 33, size=S)
    qs[:96] = 32
    ins = H.random_step_inputs(rng, S, 0, cfg, qs=qs)
    off = ins["seg_off"]
    ins["deadline_us"][off[100]] += 1 << 28
    ins["eff_prompt"][off[200]] = (1 << 17) + 7
    ctx = asc.Context(cfg, 0)
    got = ctx.schedule_step(dev(ins))
    torch.cuda.synchronize()
    exp = O.schedule_step(cfg, **ins)
    for k in ("admit_cnt", "offload_cnt", "drop_cnt", "batch_lat_us"):
        assert np.array_equal(got[k].cpu().numpy()[:S], exp[k][:S]), k
    ctx.close()
    print("ok step lanes", int(qs.sum()), "entries")


def fit_case():
    from gen import records as RC
    rec = RC.make_records(3, [40, 9000, 20000])
    ctx = asc.Context(P.config(), 0)
    ctx.fit_perf(dev(rec), 1e-8, errors=True)
    torch.cuda.synchronize()
    ctx.close()
    print("ok fit")


def latency_case():
    ctx = asc.Context(P.config(), 0)
    g = torch.Generator(device="cuda:0").manual_seed(1)
    F = torch.randint(0, 1 << 50, (100_000,), device="cuda:0", generator=g)
    M = torch.randint(0, 1 << 40, (100_000,), device="cuda:0", generator=g)
    ctx.latency(F, M)
    torch.cuda.synchronize()
    ctx.close()
    print("ok latency")


if __name__ == "__main__":
    which = sys.argv[1:] or ["sim", "step", "fit", "latency"]
    if "sim" in which:
        sim_case("config1", 200)
        sim_case("config2", 2000, max_traces=3)
        sim_case("config4", 3000)
    if "step" in which:
        step_case()
        lane_case()
    if "fit" in which:
        fit_case()
    if "latency" in which:
        latency_case()
    print("sanitize_run done")
