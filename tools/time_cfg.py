"""Time asc_simulate_batch on a named workload (optionally fewer requests / traces)."""
import os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from gen import presets as P
from paper_2504_20828_b200 import asc
name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
traces = int(sys.argv[3]) if len(sys.argv) > 3 else None
t0 = time.time()
cfg, b = P.workload(name, n=n, max_traces=traces)
print(f"{name}: T={b.T} R={b.R} gen {time.time()-t0:.1f}s", flush=True)
ctx = asc.Context(cfg, 0)
tr = asc.batch_arrays(b, "cuda:0")
for rep in range(2):
    t = time.time()
    out = ctx.simulate_batch(tr)
    ms = ctx.last_kernel_ms()
    d = int(out["decisions"].sum()); ev = int(out["evaluations"].sum())
    st = out["status"][:b.R].cpu().numpy() & 3
    print(f"  kernel {ms:.1f} ms decisions {d} ({d/ms*1e3:.3e}/s) evaluations {ev} "
          f"({ev/ms*1e3:.3e}/s) completed {int((st==1).sum())}/{b.R}", flush=True)
