"""Goodput vs QPS: Ascendra (2 LP + 1 HP) against the vLLM-like and Sarathi-like baselines (3
homogeneous instances) on the same synthetic traces — the shape of the paper's Fig goodput_main
(P:453-510), not its numbers (those need the A100 testbed and real datasets).  GPU only.
usage: goodput_sweep.py [shape] [n] [seeds] [j,j,...]   (QPS = j / 8)"""
import json, os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from gen import presets as P
from gen import traces as TR
from paper_2504_20828_b200 import asc

shape = sys.argv[1] if len(sys.argv) > 1 else "sharegpt"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
seeds = int(sys.argv[3]) if len(sys.argv) > 3 else 16
js = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [8, 32, 64, 96, 128, 160, 192, 256]
ttft, tbt = P.SLO[shape]
pts = [(qi * seeds + sd, j, 1, 1) for qi, j in enumerate(js) for sd in range(seeds)]
b = TR.grid_batch(pts, n, shape, ttft, tbt)
base = P.config(topo=P.topology(lp_token_budget=65536 if shape == "longbench" else 8192))
systems = {"ascendra_2L1H": base}
v = {k: dict(x) for k, x in base.items()}
v["topo"].update(n_lp=3, n_hp=0)
v["flags"].update(scheduler=P.SCHEDULER["vllm"], offload=0, tickets=0, policy=P.POLICY["FCFS"])
systems["vllm_3x"] = v
sa = {k: dict(x) for k, x in v.items()}
sa["flags"].update(scheduler=P.SCHEDULER["sarathi"], chunk_tokens=512)
systems["sarathi_3x"] = sa
res = {"shape": shape, "requests_per_trace": n, "seeds": seeds, "qps": [j / 8 for j in js], "goodput": {}}
tr = asc.batch_arrays(b, "cuda:0")
for name, cfg in systems.items():
    ctx = asc.Context(cfg, 0)
    out = ctx.simulate_batch(tr)
    res.setdefault("kernel_ms", {})[name] = ctx.last_kernel_ms()
    good, total = ctx.goodput(tr, out)
    g = good[:b.T].cpu().numpy().view(np.uint64).astype(np.float64)
    t = total[:b.T].cpu().numpy().view(np.uint64).astype(np.float64)
    per = [(g[i * seeds:(i + 1) * seeds].sum() / t[i * seeds:(i + 1) * seeds].sum()) for i in range(len(js))]
    res["goodput"][name] = [round(x, 4) for x in per]
    ctx.close()
print(json.dumps(res))
