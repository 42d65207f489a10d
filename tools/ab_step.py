"""A/B of asc_schedule_step builds on the row-S shapes in ONE process (GPU box): inputs are generated
once, then each library (a separate ctypes handle per .so path) is timed in alternation.
usage: python tools/ab_step.py lib1.so lib2.so ... [--shapes 1000000x32,4096x10000] [--rounds 3]"""
import argparse
import importlib
import importlib.util
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from gen import presets as P  # noqa: E402
import helpers as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--shapes", default="1000000x32,4096x10000")
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()

mods = []
for i, lib in enumerate(a.libs):  # one module object (and ctypes handle) per build
    os.environ["ASC_LIB"] = os.path.abspath(lib)
    spec = importlib.util.spec_from_file_location(f"asc_ab{i}", os.path.join(ROOT, "paper_2504_20828_b200", "asc.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    m.lib()  # bind this handle now (ASC_LIB is read at import)
    mods.append(m)

cfg = P.config()
for shp in a.shapes.split(","):
    S, Q = (int(x) for x in shp.split("x"))
    rng = np.random.default_rng(123)
    ins = H.random_step_inputs(rng, S, 0, cfg, qs=np.full(S, Q))
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in ins.items()}
    d["Q"] = S * Q
    ctxs = [m.Context(cfg, 0) for m in mods]
    ref = None
    for c in ctxs:  # warm-up + outputs must agree across builds
        for _ in range(3):
            out = c.schedule_step(d, want_prefill=False)
        sig = tuple(int(out[k].sum()) for k in ("admit_cnt", "offload_cnt", "drop_cnt"))
        ref = ref or sig
        assert sig == ref, (sig, ref)
    res = {lib: [] for lib in a.libs}
    for _ in range(a.rounds):
        for lib, c in zip(a.libs, ctxs):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k1, k2 = [], []
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.reps):
                c.schedule_step(d, want_prefill=False)
                k1.append(c.last_kernel_ms())
                k2.append(c.last_kernel2_ms())
            e1.record()
            torch.cuda.synchronize()
            res[lib].append((e0.elapsed_time(e1) / a.reps, float(np.mean(k1)), float(np.mean(k2))))
    for lib in a.libs:
        r = np.array(res[lib])
        print(f"{shp} {os.path.basename(lib)}: call {r[:,0].min():.4f}-{r[:,0].max():.4f} ms  "
              f"k1 {r[:,1].min():.4f} ms  kernel2 {r[:,2].min():.4f}-{r[:,2].max():.4f} ms")
    for c in ctxs:
        c.close()
