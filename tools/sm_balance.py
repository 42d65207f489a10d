"""Debug: per-SM finish times of the config-3 grid (library built with -DASC_DEBUG_CLOCK: evaluations
carry (smid << 48) | finish ns).  Shows how long each SM idles before the kernel ends."""
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
ms = ctx.last_kernel_ms()
e = out["evaluations"][:b.T].cpu().numpy().view(np.uint64)
sm = (e >> 48).astype(np.int64)
t = (e & ((1 << 48) - 1)).astype(np.int64)
t = (t - t.min()) / 1e6
print("kernel ms", ms, "first finish offset 0, last", t.max())
last = np.array([t[sm == s].max() for s in np.unique(sm)])
cnt = np.array([(sm == s).sum() for s in np.unique(sm)])
print("SMs", len(last), "traces per SM min/max", cnt.min(), cnt.max())
print("per-SM last finish (ms after first trace finish): min %.1f p10 %.1f median %.1f p90 %.1f max %.1f" %
      (last.min(), np.percentile(last, 10), np.median(last), np.percentile(last, 90), last.max()))
print("mean idle tail per SM: %.1f ms of %.1f" % ((last.max() - last).mean(), ms))
