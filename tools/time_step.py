"""Quick timing of asc_schedule_step on the row-S microbenchmark shapes."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from gen import presets as P
from paper_2504_20828_b200 import asc
import helpers as H
peak = 6555.2
for S, Q in ((4096, 10000), (64, 1000000), (1000000, 32), (1, 1), (100000, 32)):
    rng = np.random.default_rng(123)
    cfg = P.config()
    ins = H.random_step_inputs(rng, S, 0, cfg, qs=np.full(S, Q))
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in ins.items()}
    d["Q"] = S * Q
    ctx = asc.Context(cfg, 0)
    for _ in range(3):
        out = ctx.schedule_step(d, want_prefill=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    k1 = []; k2 = []
    for _ in range(5):
        out = ctx.schedule_step(d, want_prefill=False); k1.append(ctx.last_kernel_ms()); k2.append(ctx.last_kernel2_ms())
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    nout = int(out["admit_cnt"].sum() + out["offload_cnt"].sum() + out["drop_cnt"].sum())
    byts = 13 * S * Q + 4 * nout + S * 56
    print(f"S={S} Q={Q}: call {ms:.3f} ms k1 {np.mean(k1):.3f} ms  {byts/ms/1e6:.0f} GB/s = {byts/ms/1e6/peak*100:.1f}% of HBM; k1-only {13*S*Q/np.mean(k1)/1e6:.0f} GB/s; kernel2 {np.mean(k2):.4f} ms")
    ctx.close()
