"""Quick timing of asc_simulate_batch on config3 (optionally fewer requests per trace)."""
import sys, os, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from gen import presets as P
from paper_2504_20828_b200 import asc
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
cfg, b = P.workload("config3", n=n)
ctx = asc.Context(cfg, 0)
tr = asc.batch_arrays(b, "cuda:0")
for rep in range(2):
    t = time.time()
    out = ctx.simulate_batch(tr)
    ms = ctx.last_kernel_ms()
    d = int(out["decisions"].sum())
    print(f"n={n} kernel {ms:.1f} ms wall {time.time()-t:.2f}s decisions {d} -> {d/ms*1e3:.3e}/s", flush=True)
