"""Configuration presets and workload definitions (INPUT DATA ONLY — no method arithmetic).

Plain dicts consumed by both the oracle wrapper (oracle/oracle.py) and the
product binding (paper_2504_20828_b200/asc.py); each side marshals them into
its own struct.  Sources are cited per field; values the paper never prints
are marked "reading" and listed in DESIGN.md §Readings.
"""
from . import traces as _tr

POLICY = {"EDF_LAXITY": 0, "EDF_DEADLINE": 1, "SJF": 2, "LJF": 3, "FCFS": 4, "WEIGHTED": 5}
# Ascendra (LP/HP) or a baseline scheduler on homogeneous instances
SCHEDULER = {"ascendra": 0, "vllm": 1, "sarathi": 2}

# Mistral-7B public shape (the paper prints none; h and L match P:100's 4096 x 32).
MISTRAL7B = dict(h=4096, n=32, s=128, n_kv=8, m=14336, L=32,
                 b=128,          # attention block size: reading G15 (paper silent)
                 dtype_bytes=2,  # FP16
                 tp=1)

# TINY-LINEAR: makes lat(s) = M = 6 + 15*sum(p) + 12*B_d + 2*sum(lhat) exactly (SURVEY c.11).
TINY = dict(h=1, n=1, s=1, n_kv=1, m=1, L=1, b=1 << 20, dtype_bytes=1, tp=1)

# A100 caps; coefficients (0,1,0,0,3e-4): SPEC S:189 default, not a paper value (reading G16).
PERF_ROOFLINE = dict(c=(0.0, 1.0, 0.0, 0.0, 3e-4), F_H=312e12, M_H=2e12)
# Reading G16 (calibrated): t = 8 tM + 3 tF + 5 ms -- memory-bound work at 1/8 and compute at 1/3 of
# the A100 caps, no overlap, a 5 ms per-iteration overhead.  Invented (the paper prints no C1..C5),
# tuned ONCE on the CPU oracle (tools/calibrate_preset.py, profiles/r02_calibrate_preset.txt) so that
# the 2L1H ShareGPT-shaped goodput cliff falls inside config 3's QPS range 0.5-8 (P:505 reports
# saturation at 2.55-2.8 QPS on 3x A100; P:451/P:510 centre the axes on the ~90%-goodput knee).
# Parity-neutral: it changes what is simulated, not whether the GPU equals the oracle.
PERF_CALIBRATED = dict(c=(0.0, 0.0, 8.0, 3.0, 5e-3), F_H=312e12, M_H=2e12)
PERF = {"roofline": PERF_ROOFLINE, "calibrated": PERF_CALIBRATED}
# t = M/M_H exactly with M_H = 1: latency in seconds equals the byte count M.
PERF_TINY = dict(c=(0.0, 0.0, 1.0, 0.0, 0.0), F_H=1.0, M_H=1.0)


def topology(n_lp=2, n_hp=1, block_tokens=16, kv_blocks_lp=25000, kv_blocks_hp=25000,
             lp_max_batch=128, lp_token_budget=8192, hp_token_budget=8192):
    # 16 tok/block (reading G32), 25,000 blocks, batch 128, budgets (reading G38)
    return dict(n_lp=n_lp, n_hp=n_hp, block_tokens=block_tokens, kv_blocks_lp=kv_blocks_lp,
                kv_blocks_hp=kv_blocks_hp, lp_max_batch=lp_max_batch,
                lp_token_budget=lp_token_budget, hp_token_budget=hp_token_budget)


def flags(policy="EDF_LAXITY", offload=1, tickets=1, elastic=1, drop=0,
          offload_margin_us=0, offload_delay_us=0, hist_default_tokens=256, scheduler="ascendra",
          chunk_tokens=512, offload_rule=0, key_weights=(1, -1, 0)):
    # chunk_tokens: Sarathi-like per-batch token budget (reading G47; 512 as in SPEC S:398)
    # EDF default; offload (§5.3); tickets (§6.1); elastic (§6.2); drop off (§6.3 is a mode)
    return dict(policy=POLICY[policy] if isinstance(policy, str) else int(policy),
                offload=offload, tickets=tickets, elastic=elastic, drop=drop,
                offload_margin_us=offload_margin_us, offload_delay_us=offload_delay_us,
                hist_default_tokens=hist_default_tokens,
                scheduler=SCHEDULER[scheduler] if isinstance(scheduler, str) else int(scheduler),
                chunk_tokens=chunk_tokens, offload_rule=offload_rule, key_weights=tuple(key_weights))


def config(arch=None, perf=None, topo=None, flg=None):
    return dict(arch=dict(arch or MISTRAL7B), perf=dict(perf or PERF_ROOFLINE),
                topo=dict(topo or topology()), flags=dict(flg or flags()))


# Table 2 SLOs, microseconds.
SLO = {"sharegpt": (1_000_000, 150_000), "longbench": (2_500_000, 150_000)}


# Perf preset per workload: the QPS grids of configs 2, 3 and 5 (0.5-8 QPS) are centred on the
# calibrated preset's saturation point; configs 1 and 4 keep the roofline preset (config 4's QPS is
# frozen at 2x the roofline 2L1H LongBench saturation, so its queues are already deep).
DEFAULT_PERF = {"config1": "roofline", "config2": "calibrated", "config3": "calibrated",
                "config4": "roofline", "config5": "calibrated"}


def workload(name, n=None, max_traces=None, base_seed=1, select=None, perf=None):
    """BASELINE.json configs -> (asc config dict, TraceBatch).  DESIGN.md §Workloads.
    select: optional grid-point indices (e.g. one rank's shard), generated alone and in that order.
    perf: "roofline" | "calibrated" (default DEFAULT_PERF[name])."""
    pf = PERF[perf or DEFAULT_PERF.get(name, "roofline")]
    if name == "config1":      # 1 trace, 1L1H, 200 req, QPS 2
        cfg = config(topo=topology(n_lp=1, n_hp=1))
        pts = [(0, 16, 16, 16)]
        n = n or 200
        shape = "sharegpt"
    elif name == "config2":    # 8 traces (QPS 1..8), 2L1H, 10k req
        cfg = config()
        pts = [(j - 1, 8 * j, 16, 16) for j in range(1, 9)]
        n = n or 10_000
        shape = "sharegpt"
    elif name == "config3":    # 16 QPS x 16 SLO scales x 16 seeds = 4096 traces x 10k
        cfg = config()
        pts = []
        for qi in range(16):
            for si in range(16):
                for sd in range(16):
                    pts.append(((qi * 16 + si) * 16 + sd, 4 * (qi + 1), si + 1, 4))
        n = n or 10_000
        shape = "sharegpt"
    elif name == "config4":    # 1 trace, LongBench-shaped, deep queues
        cfg = config(topo=topology(lp_token_budget=65536))
        pts = [(0, 96, 16, 16)]   # QPS 12 = ~2x the oracle-measured 2L1H saturation (frozen)
        n = n or 1_000_000
        shape = "longbench"
    elif name == "config5":    # 64 QPS x 64 scales x 16 seeds = 65536 traces x 100k
        cfg = config()
        pts = []
        for qi in range(64):
            for si in range(64):
                for sd in range(16):
                    pts.append(((qi * 64 + si) * 16 + sd, qi + 1, si + 1, 16))
        n = n or 100_000
        shape = "sharegpt"
    else:
        raise KeyError(name)
    cfg["perf"] = dict(pf)
    if max_traces is not None:
        pts = pts[:max_traces]
    if select is not None:
        pts = [pts[int(i)] for i in select]
    ttft, tbt = SLO[shape]
    return cfg, _tr.grid_batch(pts, n, shape, ttft, tbt, base_seed)
