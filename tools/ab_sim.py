"""A/B of asc_simulate_batch builds on config 3 in ONE process (GPU box): the traces are generated
once, then each library (a separate ctypes handle per .so path) is timed in alternation; digests and
decision counts must agree across builds.
usage: python tools/ab_sim.py lib1.so lib2.so ... [--n 10000] [--rounds 3] [--workload config3]"""
import argparse
import importlib.util
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from gen import presets as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--n", type=int, default=10000)
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--workload", default="config3")
ap.add_argument("--nodigest", action="store_true", help="compare decisions only (experimental builds)")
a = ap.parse_args()

mods = []
for i, lib in enumerate(a.libs):  # one module object (and ctypes handle) per build
    os.environ["ASC_LIB"] = os.path.abspath(lib)
    spec = importlib.util.spec_from_file_location(f"asc_ab{i}", os.path.join(ROOT, "paper_2504_20828_b200", "asc.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    m.lib()
    mods.append(m)

cfg, b = P.workload(a.workload, n=a.n)
ctxs = [m.Context(cfg, 0) for m in mods]
trs = [m.batch_arrays(b, "cuda:0") for m in mods]
ref = None
for c, tr in zip(ctxs, trs):
    out = c.simulate_batch(tr)
    sig = (int(out["decisions"].sum()), 0 if a.nodigest else int(out["digest"].sum()))
    ref = ref or sig
    assert sig == ref, (sig, ref)
res = {lib: [] for lib in a.libs}
for _ in range(a.rounds):
    for lib, c, tr in zip(a.libs, ctxs, trs):
        c.simulate_batch(tr)
        res[lib].append(c.last_kernel_ms())
for lib in a.libs:
    r = np.array(res[lib])
    print(f"{a.workload} n={a.n} {os.path.basename(lib)}: kernel {r.min():.1f}-{r.max():.1f} ms (median {np.median(r):.1f})",
          flush=True)
