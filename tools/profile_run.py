"""Run one kernel of interest once after warm-up (for ncu captures; never a bench number)."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from gen import presets as P  # noqa: E402
from paper_2504_20828_b200 import asc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("what", choices=["sim", "step", "fit"])
ap.add_argument("--traces", type=int, default=512)
ap.add_argument("--n", type=int, default=1000)
ap.add_argument("--S", type=int, default=4096)
ap.add_argument("--Q", type=int, default=10000)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--workload", default="config3")
ap.add_argument("--select", default=None, help="comma-separated trace indices (sim)")
a = ap.parse_args()
if a.what == "sim":
    cfg, b = P.workload(a.workload, n=a.n)
    if a.select:
        b = b.subset([int(x) for x in a.select.split(",")])
    elif a.traces < b.T:
        b = b.subset(np.linspace(0, b.T - 1, a.traces).round().astype(int))
    ctx = asc.Context(cfg, 0)
    tr = asc.batch_arrays(b, "cuda:0")
    for _ in range(a.reps):
        out = ctx.simulate_batch(tr)
        print("sim ms", ctx.last_kernel_ms(), "decisions", int(out["decisions"].sum()))
elif a.what == "fit":
    from gen import records as RC
    rec = RC.make_records(21, [65536] * 1024)
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in rec.items()}
    ctx = asc.Context(P.config(), 0)
    for _ in range(a.reps):
        ctx.fit_perf(d, 1e-8, errors=False)
        print("fit ms", ctx.last_kernel_ms())
else:
    import helpers as H
    rng = np.random.default_rng(123)
    cfg = P.config()
    ins = H.random_step_inputs(rng, a.S, 0, cfg, qs=np.full(a.S, a.Q))
    dins = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in ins.items()}
    ctx = asc.Context(cfg, 0)
    for _ in range(a.reps):
        out = ctx.schedule_step(dins, want_prefill=False)
        print("k1 ms", ctx.last_kernel_ms())
torch.cuda.synchronize()
