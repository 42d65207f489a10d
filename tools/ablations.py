"""Ablations of §8.3-8.5 on the GPU (row f4, Fig ablation_eb_val, Fig drop):
reorder policy (EDF vs SJF vs FCFS vs LJF), elastic HP batch on/off, dropping
requests past their TTFT SLO under overload; 2L1H, ShareGPT-shaped, 16 seeds per point.
usage: ablations.py [n] [seeds] [j,j,...]   (QPS = j / 8)"""
import json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from gen import presets as P
from gen import traces as TR
from paper_2504_20828_b200 import asc

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
seeds = int(sys.argv[2]) if len(sys.argv) > 2 else 16
js = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [512, 768, 1024, 1280]
ttft, tbt = P.SLO["sharegpt"]
pts = [(qi * seeds + sd, j, 1, 1) for qi, j in enumerate(js) for sd in range(seeds)]
b = TR.grid_batch(pts, n, "sharegpt", ttft, tbt)
tr = asc.batch_arrays(b, "cuda:0")
variants = {f"policy_{p}": dict(policy=p) for p in ("EDF_LAXITY", "EDF_DEADLINE", "SJF", "FCFS", "LJF")}
variants["elastic_off"] = dict(elastic=0)
variants["drop_on"] = dict(drop=1)
variants["offload_off"] = dict(offload=0)
variants["tickets_off"] = dict(tickets=0)
res = {"qps": [j / 8 for j in js], "requests_per_trace": n, "seeds": seeds, "goodput": {},
       "dropped_frac": {}}
for name, fl in variants.items():
    ctx = asc.Context(P.config(flg=P.flags(**fl)), 0)
    out = ctx.simulate_batch(tr)
    good, total = ctx.goodput(tr, out)
    g = good[:b.T].cpu().numpy().view(np.uint64).astype(np.float64)
    t = total[:b.T].cpu().numpy().view(np.uint64).astype(np.float64)
    st = out["status"][:b.R].cpu().numpy().view(np.uint32) & 3
    ctx.close()
    res["goodput"][name] = [round(float(g[i * seeds:(i + 1) * seeds].sum() / t[i * seeds:(i + 1) * seeds].sum()), 4)
                            for i in range(len(js))]
    if fl.get("drop"):
        off = b.trace_off
        res["dropped_frac"][name] = [round(float((st[off[i * seeds]:off[(i + 1) * seeds]] == 2).mean()), 4)
                                     for i in range(len(js))]
print(json.dumps(res))
