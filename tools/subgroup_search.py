"""Subgroup configuration search (row f3, Fig scale_fig): for a pool of K
instances, every Ascendra split n_lp + n_hp = K (n_lp >= 1) runs as one more grid axis of a
single asc_simulate_batch call (per-trace topology), beside the baselines on K homogeneous
instances; reports goodput per QPS and the best configuration.  GPU only.
usage: subgroup_search.py [shape] [K] [n] [seeds] [j,j,...]   (QPS = j / 8)"""
import json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from gen import presets as P
from gen import traces as TR
from paper_2504_20828_b200 import asc

shape = sys.argv[1] if len(sys.argv) > 1 else "sharegpt"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
seeds = int(sys.argv[4]) if len(sys.argv) > 4 else 16
js = [int(x) for x in sys.argv[5].split(",")] if len(sys.argv) > 5 else [256, 512, 768, 1024, 1280]
ttft, tbt = P.SLO[shape]
splits = [(K - h, h) for h in range(0, K)]  # (n_lp, n_hp), n_lp >= 1
pts = [(qi * seeds + sd, j, 1, 1) for qi, j in enumerate(js) for sd in range(seeds)]
b = TR.grid_batch(pts, n, shape, ttft, tbt)
tok = 65536 if shape == "longbench" else 8192
res = {"shape": shape, "pool": K, "requests_per_trace": n, "seeds": seeds, "qps": [j / 8 for j in js],
       "goodput": {}, "kernel_ms": {}}

def run(cfg, nl=None, nh=None):
    tr = asc.batch_arrays(b, "cuda:0")
    # the whole topology axis in one call: traces repeated once per split
    ctx = asc.Context(cfg, 0)
    out = ctx.simulate_batch(tr, n_lp=nl, n_hp=nh)
    ms = ctx.last_kernel_ms()
    good, total = ctx.goodput(tr, out)
    ctx.close()
    g = good[:b.T].cpu().numpy().view(np.uint64).astype(np.float64)
    t = total[:b.T].cpu().numpy().view(np.uint64).astype(np.float64)
    return g, t, ms

# Ascendra: the split axis in one call (the batch repeated once per split)
rep = TR.make_batch([b.trace(t)[:3] for _ in splits for t in range(b.T)],
                    list(b.ttft_slo_us) * len(splits), list(b.tbt_slo_us) * len(splits))
nl = np.repeat(np.array([s[0] for s in splits], np.int32), b.T)
nh = np.repeat(np.array([s[1] for s in splits], np.int32), b.T)
cfg = P.config(topo=P.topology(n_lp=K - 1, n_hp=1, lp_token_budget=tok))
tr = asc.batch_arrays(rep, "cuda:0")
ctx = asc.Context(cfg, 0)
out = ctx.simulate_batch(tr, n_lp=torch.from_numpy(nl).cuda(), n_hp=torch.from_numpy(nh).cuda())
res["kernel_ms"]["ascendra_all_splits"] = ctx.last_kernel_ms()
good, total = ctx.goodput(tr, out)
ctx.close()
g = good[:rep.T].cpu().numpy().view(np.uint64).astype(np.float64)
t = total[:rep.T].cpu().numpy().view(np.uint64).astype(np.float64)
for si, (l, h) in enumerate(splits):
    gs, ts = g[si * b.T:(si + 1) * b.T], t[si * b.T:(si + 1) * b.T]
    res["goodput"][f"ascendra_{l}L{h}H"] = [round(float(gs[i * seeds:(i + 1) * seeds].sum() / ts[i * seeds:(i + 1) * seeds].sum()), 4) for i in range(len(js))]
for name in ("vllm", "sarathi"):
    c = P.config(topo=P.topology(n_lp=K, n_hp=0, lp_token_budget=tok),
                 flg=P.flags(policy="FCFS", offload=0, tickets=0, scheduler=name))
    gg, tt, ms = run(c)
    res["kernel_ms"][name] = ms
    res["goodput"][f"{name}_{K}x"] = [round(float(gg[i * seeds:(i + 1) * seeds].sum() / tt[i * seeds:(i + 1) * seeds].sum()), 4) for i in range(len(js))]
res["best"] = [max(res["goodput"], key=lambda k: res["goodput"][k][i]) for i in range(len(js))]
print(json.dumps(res))
