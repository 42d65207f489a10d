"""Debug: per-trace finish times (needs a library built with -DASC_DEBUG_CLOCK)."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from gen import presets as P
from paper_2504_20828_b200 import asc
cfg, b = P.workload("config3")
ctx = asc.Context(cfg, 0)
tr = asc.batch_arrays(b, "cuda:0")
out = ctx.simulate_batch(tr)
t = (out["evaluations"][:b.T].cpu().numpy().view(np.uint64) & ((1 << 48) - 1)).astype(np.int64)
d = out["decisions"][:b.T].cpu().numpy()
t = (t - t.min()) / 1e6  # ns -> ms after the first finisher
order = np.argsort(-t)
print("kernel ms", ctx.last_kernel_ms())
for i in order[:15]:
    print(f"trace {i:5d} {b.labels[i]:28s} finish {t[i]:8.1f} ms decisions {d[i]}")
qps = b.qps_j
for j in sorted(set(qps.tolist())):
    m = qps == j
    print(f"qps {j/8:5.2f}: mean finish {t[m].mean():7.1f} ms max {t[m].max():7.1f} ms mean decisions {d[m].mean():.0f}")
