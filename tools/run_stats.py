"""Debug: decode-run statistics per QPS (needs a library built with -DASC_DEBUG_RUNS)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from gen import presets as P
from paper_2504_20828_b200 import asc
cfg, b = P.workload("config3")
ctx = asc.Context(cfg, 0)
out = ctx.simulate_batch(asc.batch_arrays(b, "cuda:0"))
ev = out["evaluations"][:b.T].cpu().numpy().astype(np.int64)
d = out["decisions"][:b.T].cpu().numpy()
# per trace: sum over runs of (1<<32) + J, plus the ordinary evaluations (< 2^32)
inv = ev >> 32
low = ev & 0xffffffff  # run decisions + ordinary evaluations (mod 2^32)
for j in sorted(set(b.qps_j.tolist())):
    m = b.qps_j == j
    print(f"qps {j/8:5.2f}: decisions/trace {d[m].mean():9.0f}  runs/trace {inv[m].mean():9.0f}  "
          f"run-len {((low[m]).sum()/max(inv[m].sum(),1)):6.1f}")
print("total runs", inv.sum(), "decisions", d.sum())
