"""asc_goodput (row a8) on config 3 outcomes: event-timed kernel ms and achieved bandwidth."""
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
res = {k: torch.empty(b.T, dtype=torch.int64, device="cuda:0") for k in ("good", "total")}
for _ in range(3):
    ctx.goodput(tr, out, res=res)
ms = []
for _ in range(10):
    ctx.goodput(tr, out, res=res)
    ms.append(ctx.last_kernel_ms())
k = float(np.median(ms))
byts = 32 * b.R + 16 * b.T + 8 * (b.T + 1) + 16 * b.T
print(f"goodput kernel {k * 1e3:.0f} us, {byts / k / 1e6:.0f} GB/s (32 B/request), good {int(res['good'].sum())}/{int(res['total'].sum())}")
