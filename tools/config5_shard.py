"""Config 5 on one GPU: shard r of W of the 65,536-trace x 100k-request grid (traces i = r mod W,
as bench.py / dist.py shard it), timed with CUDA events; a few traces of the shard re-run on the
CPU oracle for parity.  usage: config5_shard.py [W=16] [r=0] [n=100000] [oracle_traces=4]"""
import os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from gen import presets as P
from paper_2504_20828_b200 import asc
from paper_2504_20828_b200 import dist as D

W = int(sys.argv[1]) if len(sys.argv) > 1 else 16
r = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 100_000
n_or = int(sys.argv[4]) if len(sys.argv) > 4 else 4
t0 = time.time()
cfg, full = P.workload("config5", n=1)
idx = D.shard(full.T, r, W)
cfg, b = P.workload("config5", n=n, select=idx)
print(f"config5 shard {r}/{W}: T={b.T} R={b.R} (gen {time.time() - t0:.0f} s)", flush=True)
ctx = asc.Context(cfg, 0)
tr = asc.batch_arrays(b, "cuda:0")
out = ctx.simulate_batch(tr)
good, total = ctx.goodput(tr, out)
for rep in range(2):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.simulate_batch(tr, out=out)
    sim_ms = ctx.last_kernel_ms()
    good, total = ctx.goodput(tr, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    dec = int(out["decisions"][:b.T].sum())
    st = out["status"][:b.R].cpu().numpy().view(np.uint32) & 3
    fin = int((st != 0).sum())
    g = int(good[:b.T].cpu().numpy().view(np.uint64).sum())
    tot = int(total[:b.T].cpu().numpy().view(np.uint64).sum())
    print(f"  step {ms:.0f} ms (sim kernel {sim_ms:.0f} ms): {dec / ms * 1e3:.3e} decisions/s, "
          f"{fin / ms * 1e3:.3e} simulated req/s, goodput {g}/{tot}", flush=True)
if n_or > 0:
    from oracle import oracle as O
    pick = np.linspace(0, b.T - 1, n_or).round().astype(int).tolist()
    sub = b.subset(pick)
    t0 = time.time()
    exp = O.simulate_batch(cfg, sub, nthreads=n_or)
    dig = out["digest"][:b.T].cpu().numpy().view(np.uint64)[pick]
    decs = out["decisions"][:b.T].cpu().numpy()[pick]
    ok = np.array_equal(dig, exp["digest"]) and np.array_equal(decs, exp["decisions"])
    print(f"  oracle parity on traces {pick}: {'OK' if ok else 'MISMATCH'} ({time.time() - t0:.0f} s)")
ctx.close()
