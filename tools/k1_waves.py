"""k1 duration vs segment count at Q = 10,000 (tail/wave effects of the one-warp-per-task grid)."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from gen import presets as P
from paper_2504_20828_b200 import asc
import helpers as H
Q = 10000
cfg = P.config()
for S in [int(a) for a in (sys.argv[1:] or "592 1184 1776 2368 2960 3552 4096 4736".split())]:
    rng = np.random.default_rng(123)
    ins = H.random_step_inputs(rng, S, 0, cfg, qs=np.full(S, Q))
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in ins.items()}
    d["Q"] = S * Q
    ctx = asc.Context(cfg, 0)
    for _ in range(3):
        ctx.schedule_step(d, want_prefill=False)
    k1 = []
    for _ in range(10):
        ctx.schedule_step(d, want_prefill=False); k1.append(ctx.last_kernel_ms())
    ms = float(np.median(k1))
    print(f"S={S}: k1 {ms*1e3:.1f} us  {ms*1e3/S*1000:.2f} ns/segment  {13*S*Q/ms/1e6:.0f} GB/s")
    ctx.close()
