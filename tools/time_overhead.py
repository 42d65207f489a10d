"""Fixed per-call cost of asc_schedule_step (GPU box): the Python binding's marshalling, the C call
(host checks, launches, error sync), and the device time of the launches (S = 1, Q = 1)."""
import ctypes as C, os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from gen import presets as P
from paper_2504_20828_b200 import asc
import helpers as H
cfg = P.config()
for S, Q, strm in ((1, 1, None), (1, 1, 'torch'), (1000000, 32, None), (1000000, 32, 'torch')):
    ins = H.random_step_inputs(np.random.default_rng(1), S, 0, cfg, qs=np.full(S, Q))
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in ins.items()}
    d["Q"] = S * Q
    sobj = torch.cuda.Stream() if strm else None
    ctx = asc.Context(cfg, 0, sobj)
    out = ctx.schedule_step(d, want_prefill=False)
    n = 200 if S == 1 else 20
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        ctx.schedule_step(d, want_prefill=False, out=out)
    t1 = time.perf_counter()
    i = asc.asc_step_in(S, S * Q, *[asc._ptr(d[k]) for k in ("seg_off", "now_us", "deadline_us", "eff_prompt", "flags",
                                                          "dec_count", "dec_ctx_sum", "tbt_slo_us", "budget_tokens",
                                                          "budget_blocks", "budget_reqs")])
    o = asc.asc_step_out(*[asc._ptr(out[k]) for k in ("admit_idx", "admit_cnt", "offload_idx", "offload_cnt", "drop_idx",
                                                      "drop_cnt", "batch_lat_us", "prefill_us")])
    L = asc.lib()
    t2 = time.perf_counter()
    for _ in range(n):
        L.asc_schedule_step(ctx.h, C.byref(i), C.byref(o))
    t3 = time.perf_counter()
    print(f"S={S} Q={Q} stream={strm}: python API {1e6*(t1-t0)/n:.1f} us/call, C call alone {1e6*(t3-t2)/n:.1f} us/call, "
          f"launches {ctx.last_launches()}")
    ctx.close()
