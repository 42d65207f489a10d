"""Tune the `calibrated` perf preset (reading G16) ONCE on the CPU oracle.

The paper prints no C1..C5.  With the `roofline` preset the 2L1H ShareGPT-shaped
cliff sits at ~100 QPS, far outside config 3's QPS grid 0.5-8, so that grid never queues.  This
script sweeps t = C3 tM + C4 tF + C5 (no overlap of memory and compute) and prints, per candidate,
goodput / evaluations per request / decisions per request along QPS at SLO scale 1; then the
config-3 goodput surface (QPS x SLO scale) for the chosen preset.  Oracle only (test
infrastructure); the result is frozen in gen/presets.py as PERF_CALIBRATED.
usage: calibrate_preset.py [search|grid]"""
import itertools
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from gen import presets as P  # noqa: E402
from gen import traces as TR  # noqa: E402
from oracle import oracle as O  # noqa: E402

CORES = os.cpu_count() or 1


def search(js=(8, 16, 24, 32, 40, 48, 56, 64), seeds=4, n=2000):
    pts = [(qi * seeds + sd, j, 1, 1) for qi, j in enumerate(js) for sd in range(seeds)]
    b = TR.grid_batch(pts, n, "sharegpt", *P.SLO["sharegpt"])
    print("QPS " + " ".join(f"{j / 8:g}" for j in js))
    for C3, C4, C5 in itertools.product((4, 6, 8, 10), (1, 2, 3, 4), (0.002, 0.005, 0.02)):
        cfg = P.config(perf=dict(c=(0, 0, C3, C4, C5), F_H=312e12, M_H=2e12))
        out = O.simulate_batch(cfg, b, nthreads=CORES)
        g, t = O.goodput(b, out)
        gp = [g[i * seeds:(i + 1) * seeds].sum() / t[i * seeds:(i + 1) * seeds].sum() for i in range(len(js))]
        ev = out["evaluations"].reshape(len(js), seeds).sum(1) / (n * seeds)
        dec = out["decisions"].reshape(len(js), seeds).sum(1) / (n * seeds)
        print(f"C=(0,0,{C3},{C4},{C5}): goodput " + " ".join(f"{x:.2f}" for x in gp)
              + " | eval/req " + " ".join(f"{x:.0f}" for x in ev)
              + " | dec/req " + " ".join(f"{x:.1f}" for x in dec), flush=True)


def grid(n=10_000, seeds=2, scales=(1, 2, 4, 8, 16)):
    pts = [((qi * 16 + si) * 16 + sd, 4 * (qi + 1), si, 4) for qi in range(16) for si in scales
           for sd in range(seeds)]
    b = TR.grid_batch(pts, n, "sharegpt", *P.SLO["sharegpt"])
    cfg = P.config(perf=P.PERF_CALIBRATED)
    t0 = time.time()
    out = O.simulate_batch(cfg, b, nthreads=CORES)
    dt = time.time() - t0
    g, t = O.goodput(b, out)
    G = (g.astype(float) / t).reshape(16, len(scales), seeds).mean(2)
    ev = out["evaluations"].reshape(16, len(scales), seeds).sum(2) / (n * seeds)
    dec = out["decisions"].reshape(16, len(scales), seeds).sum(2) / (n * seeds)
    k1 = scales.index(4)
    print(f"preset {P.PERF_CALIBRATED['c']}: {len(pts)} traces x {n} req, oracle {dt:.1f} s on {CORES} threads")
    print("QPS   " + " ".join(f"scale {s / 4:<5g}" for s in scales) + "   eval/req@1  dec/req@1")
    for qi in range(16):
        print(f"{(qi + 1) / 2:4.1f}  " + " ".join(f"{G[qi, k]:.3f}      " for k in range(len(scales)))
              + f"  {ev[qi, k1]:9.1f}  {dec[qi, k1]:8.1f}")


if __name__ == "__main__":
    (grid if (sys.argv[1:] or ["grid"])[0] == "grid" else search)()
