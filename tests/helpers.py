"""Shared test helpers: preset builders and fixture loaders (no method arithmetic)."""
import json
import os

import numpy as np

from gen import presets as P
from gen import traces as TR

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SEC = 1_000_000  # TINY-LINEAR fixtures are written in seconds


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def tiny_cfg(n_lp=1, n_hp=1, block_tokens=4, kv_blocks=100, lp_max_batch=4, lp_token_budget=8,
             hp_token_budget=4, policy="EDF_LAXITY", offload=1, tickets=1, elastic=0, drop=0,
             margin=0, delay=0, hist_default=256, kv_blocks_hp=None, scheduler="ascendra",
             chunk_tokens=512):
    return P.config(arch=P.TINY, perf=P.PERF_TINY,
                    topo=P.topology(n_lp=n_lp, n_hp=n_hp, block_tokens=block_tokens,
                                    kv_blocks_lp=kv_blocks,
                                    kv_blocks_hp=kv_blocks if kv_blocks_hp is None else kv_blocks_hp,
                                    lp_max_batch=lp_max_batch, lp_token_budget=lp_token_budget,
                                    hp_token_budget=hp_token_budget),
                    flg=P.flags(policy=policy, offload=offload, tickets=tickets, elastic=elastic,
                                drop=drop, offload_margin_us=margin, offload_delay_us=delay,
                                hist_default_tokens=hist_default, scheduler=scheduler,
                                chunk_tokens=chunk_tokens))


def fixture_sim(name):
    """Golden DES fixture -> (cfg, batch, expect) with times converted to microseconds."""
    g = golden(name)
    t, f = g["topology"], g["flags"]
    cfg = tiny_cfg(n_lp=t["n_lp"], n_hp=t["n_hp"], block_tokens=t["block_tokens"],
                   kv_blocks=t["kv_blocks"], lp_max_batch=t["lp_max_batch"],
                   lp_token_budget=t["lp_token_budget"], hp_token_budget=t["hp_token_budget"],
                   policy=f["policy"], offload=f["offload"], tickets=f["tickets"],
                   elastic=f["elastic"], scheduler=f.get("scheduler", "ascendra"),
                   chunk_tokens=f.get("chunk_tokens", 512))
    req = np.array(g["requests"], dtype=np.int64)
    batch = TR.make_batch([(req[:, 0] * SEC, req[:, 1], req[:, 2])], [g["ttft"] * SEC],
                          [g["tbt"] * SEC])
    return cfg, batch, g["expect"]


def w1_step_inputs(policy):
    """W1 as one stateless segment (times in microseconds)."""
    g = golden("w1_lp_formation.json")
    cfg = tiny_cfg(block_tokens=g["block_tokens"], hp_token_budget=g["hp_token_budget"],
                   policy=policy)
    w = np.array(g["waiting"], dtype=np.int64)
    ins = dict(seg_off=np.array([0, len(w)], np.int64),
               now_us=np.array([g["now"] * SEC], np.int64),
               deadline_us=(w[:, 1] + g["ttft"]) * SEC,
               eff_prompt=w[:, 2].astype(np.int32),
               flags=np.zeros(len(w), np.uint8),
               dec_count=np.array([g["decodes"]["count"]], np.int32),
               dec_ctx_sum=np.array([g["decodes"]["ctx_sum"]], np.int64),
               tbt_slo_us=np.array([g["tbt"] * SEC], np.int64),
               budget_tokens=np.array([g["budgets"]["N"]], np.int32),
               budget_blocks=np.array([g["budgets"]["M"]], np.int32),
               budget_reqs=np.array([g["budgets"]["R"]], np.int32))
    return cfg, ins, g["expect"][policy], [int(x) for x in w[:, 0]]


def random_step_inputs(rng, S, qmax, cfg, now_spread_us=3 * SEC, budgets="random", qs=None):
    """Random stateless-step segments with the shape of SURVEY §8(d) config S."""
    qs = rng.integers(0, qmax + 1, size=S) if qs is None else np.asarray(qs)
    off = np.zeros(S + 1, np.int64)
    off[1:] = np.cumsum(qs)
    Q = int(off[-1])
    now = rng.integers(10 * SEC, 20 * SEC, size=S).astype(np.int64)
    seg_of = np.repeat(np.arange(S), qs)
    tabs = TR.tables()
    eff = tabs["sharegpt_prompt"][rng.integers(0, 1 << 16, size=Q)].astype(np.int32)
    dl = now[seg_of] + rng.integers(-now_spread_us, now_spread_us + 1, size=Q)
    flags = (rng.random(Q) < 0.1).astype(np.uint8) | ((rng.random(Q) < 0.05).astype(np.uint8) << 1)
    dec = rng.integers(0, 129, size=S).astype(np.int32)
    ctx = (dec.astype(np.int64) * rng.integers(1, 3000, size=S)).astype(np.int64)
    if budgets == "random":
        N = rng.integers(0, 20000, size=S).astype(np.int32)
        M = rng.integers(0, 2000, size=S).astype(np.int32)
        R = rng.integers(0, 129, size=S).astype(np.int32)
        tbt = rng.integers(0, 400_000, size=S).astype(np.int64)
    else:
        N = np.full(S, cfg["topo"]["lp_token_budget"], np.int32)
        M = np.full(S, cfg["topo"]["kv_blocks_lp"], np.int32)
        R = np.full(S, cfg["topo"]["lp_max_batch"], np.int32)
        tbt = np.full(S, 150_000, np.int64)
    return dict(seg_off=off, now_us=now, deadline_us=dl.astype(np.int64), eff_prompt=eff,
                flags=flags, dec_count=dec, dec_ctx_sum=ctx, tbt_slo_us=tbt,
                budget_tokens=N, budget_blocks=M, budget_reqs=R)


def segment_lists(out, seg_off):
    """CSR outputs -> per-segment python lists."""
    res = []
    for s in range(len(seg_off) - 1):
        lo = int(seg_off[s])
        res.append((list(out["admit_idx"][lo:lo + int(out["admit_cnt"][s])]),
                    list(out["offload_idx"][lo:lo + int(out["offload_cnt"][s])]),
                    list(out["drop_idx"][lo:lo + int(out["drop_cnt"][s])])))
    return res
