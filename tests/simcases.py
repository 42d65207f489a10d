"""Simulation test cases shared by the oracle pins and the GPU parity tests.

Each check takes `sim(cfg, batch, req_ttft=None) -> dict` (per-request first_token_us, done_us,
prefill_start_us, status; per-trace digest, decisions) and `goodput(batch, out) -> (good, total)`,
so the same hand-worked expectations pin the oracle AND the CUDA path.
"""
import itertools

import numpy as np

import helpers as H
from gen import presets as P
from gen import traces as TR

SEC = H.SEC


def state(st):
    return np.asarray(st) & 3


def inst(st):
    return (np.asarray(st) >> 4) & 255


def npre(st):
    return (np.asarray(st) >> 12) & 0xFFFF


def check_fixture(sim, goodput, name):
    cfg, batch, exp = H.fixture_sim(name)
    out = sim(cfg, batch)
    sec = lambda a: [int(x) // SEC if x >= 0 else -1 for x in a]
    assert sec(out["first_token_us"]) == exp["first_token"]
    assert sec(out["done_us"]) == exp["done"]
    assert sec(out["prefill_start_us"]) == exp["prefill_start"]
    assert int(out["decisions"][0]) == exp["decisions"]
    st = out["status"]
    if "instance" in exp:
        assert list(inst(st)) == exp["instance"]
    if "offloaded" in exp:
        assert list((st >> 2) & 1) == exp["offloaded"]
    if "ticketed" in exp:
        assert list((st >> 3) & 1) == exp["ticketed"]
    if "preemptions" in exp:
        assert list(npre(st)) == exp["preemptions"]
    g, t = goodput(batch, out)
    assert (int(g[0]), int(t[0])) == (exp["good"], exp["total"])


def check_elastic(sim):
    g = H.golden("w5_elastic.json")
    req = np.array(g["requests"], np.int64)
    for case in g["cases"]:
        cfg = H.tiny_cfg(n_lp=1, n_hp=1, block_tokens=4, kv_blocks=100, lp_max_batch=1,
                         lp_token_budget=8, hp_token_budget=4, policy="FCFS", offload=1,
                         tickets=0, elastic=case.get("elastic", 1), margin=10 ** 15,
                         hist_default=case["hist_default"])
        b = TR.make_batch([(req[:, 0] * SEC, req[:, 1], req[:, 2])], [10 ** 4 * SEC], [10 ** 4 * SEC])
        out = sim(cfg, b)
        assert [int(x) // SEC for x in out["first_token_us"]] == case["expect_first"]


def lindley_case(rng, n):
    """FCFS degenerate case: 1 LP, no HP, batch cap 1, output 1 -> single-server FCFS queue."""
    cfg = H.tiny_cfg(n_lp=1, n_hp=0, lp_max_batch=1, lp_token_budget=64, policy="FCFS",
                     offload=0, tickets=0, kv_blocks=1000)
    arr = np.sort(rng.integers(0, 40 * n, size=n)).astype(np.int64) * SEC // 2
    p = rng.integers(1, 60, size=n)
    b = TR.make_batch([(arr, p, np.ones(n))], [10 ** 9 * SEC], [SEC])
    # Lindley recursion: start_i = max(arrival_i, end_{i-1}); end_i = start_i + (6 + 15 p_i) s
    end, prev = [], 0
    for i in range(n):
        s = max(int(arr[i]), prev)
        prev = s + (6 + 15 * int(p[i])) * SEC
        end.append(prev)
    return cfg, b, end


def single_request_case(p, o):
    cfg = H.tiny_cfg(n_lp=1, n_hp=0, lp_token_budget=p + o + 1, kv_blocks=10_000, offload=0,
                     tickets=0, policy="EDF_LAXITY")
    b = TR.make_batch([(np.array([7 * SEC]), np.array([p]), np.array([o]))], [10 ** 6 * SEC],
                      [10 ** 6 * SEC])
    first = 7 * SEC + (6 + 15 * p) * SEC
    done = first + sum((6 + 12 + 2 * (p + g)) * SEC for g in range(1, o))
    return cfg, b, first, done


def sched_case(n, p, policy, ttft_s, req_ttft_s=None):
    """n requests at t=0 on one LP with batch cap 1 and output 1 (single machine, no preemption)."""
    cfg = H.tiny_cfg(n_lp=1, n_hp=0, lp_max_batch=1, lp_token_budget=64, policy=policy,
                     offload=0, tickets=0, kv_blocks=1000)
    b = TR.make_batch([(np.zeros(n, np.int64), np.array(p), np.ones(n))], [ttft_s * SEC], [SEC])
    rt = None if req_ttft_s is None else np.array(req_ttft_s, np.int64) * SEC
    return cfg, b, rt


def check_textbook_rules(sim, goodput, rng, trials=40):
    """SPT minimises total completion time; SJF maximises on-time count under a common due date;
    EDF (Jackson's rule) minimises the maximum lateness.  Brute force over all permutations."""
    for _ in range(trials):
        n = int(rng.integers(1, 7))
        p = [int(x) for x in rng.integers(1, 50, size=n)]
        w = [6 + 15 * x for x in p]  # TINY-LINEAR prefill seconds
        perms = list(itertools.permutations(range(n)))

        def completions(order):
            t, c = 0, [0] * n
            for i in order:
                t += w[i]
                c[i] = t
            return c

        cfg, b, _ = sched_case(n, p, "SJF", 10 ** 6)
        out = sim(cfg, b)
        ttft = [int(x) // SEC for x in out["first_token_us"]]
        assert sum(ttft) == min(sum(completions(o)) for o in perms)
        due = int(rng.integers(min(w), sum(w) + 1))
        cfg, b, _ = sched_case(n, p, "SJF", due)
        out = sim(cfg, b)
        good, _ = goodput(b, out)
        assert int(good[0]) == max(sum(1 for x in completions(o) if x <= due) for o in perms)
        d = [int(x) for x in rng.integers(1, sum(w) + 1, size=n)]
        cfg, b, rt = sched_case(n, p, "EDF_DEADLINE", 1, d)
        out = sim(cfg, b, rt)
        lat = max(int(out["first_token_us"][i]) // SEC - d[i] for i in range(n))
        assert lat == min(max(c - di for c, di in zip(completions(o), d)) for o in perms)


def random_small_batch(rng, T, nmax, shape="sharegpt"):
    trs, tt, tb = [], [], []
    for t in range(T):
        n = int(rng.integers(1, nmax + 1))
        j = int(rng.integers(4, 200))
        trs.append(TR.gen_trace(int(rng.integers(1, 1 << 30)), t, shape, j, n))
        scale = int(rng.integers(1, 17))
        tt.append(1_000_000 * scale // 4)
        tb.append(150_000 * scale // 4)
    return TR.make_batch(trs, tt, tb)


def check_invariants(batch, out, cfg):
    st = out["status"]
    n_lp = cfg["topo"]["n_lp"]
    for t in range(batch.T):
        lo, hi = int(batch.trace_off[t]), int(batch.trace_off[t + 1])
        s = st[lo:hi]
        a = batch.arrival_us[lo:hi]
        f, d, ps = out["first_token_us"][lo:hi], out["done_us"][lo:hi], out["prefill_start_us"][lo:hi]
        comp = state(s) == 1
        drop = state(s) == 2
        # conservation at end of run: every request completed or dropped
        assert np.all(comp | drop)
        if not cfg["flags"]["drop"]:
            assert np.all(comp)
        # time order: arrival <= prefill start < first token <= done
        assert np.all(ps[comp] >= a[comp]) and np.all(f[comp] > ps[comp]) and np.all(d[comp] >= f[comp])
        # offloaded / ticketed requests are served on an HP, never on an LP
        ofl = ((s >> 2) & 1) == 1
        tk = ((s >> 3) & 1) == 1
        assert np.all(inst(s)[(ofl | tk) & comp] >= n_lp)
        assert not np.any(ofl & tk)


# ------------------------------------------------------------------ baselines (row f1) --------
def with_scheduler(cfg, name):
    """Same config on homogeneous baseline instances (reading G46: n_hp = 0, no offload/tickets)."""
    cfg = {k: dict(v) for k, v in cfg.items()}
    cfg["flags"]["scheduler"] = P.SCHEDULER[name]
    cfg["topo"]["n_hp"] = 0
    cfg["flags"]["offload"] = 0
    cfg["flags"]["tickets"] = 0
    return cfg


def check_vllm_fcfs_order(sim, rng, trials=4):
    """FCFS baselines never start request j's prefill before request i's when i arrived
    earlier on the same instance (checked without preemption: ample KV), round-robin routing."""
    for _ in range(trials):
        n_lp = int(rng.integers(1, 4))
        cfg = with_scheduler(P.config(topo=P.topology(n_lp=n_lp, kv_blocks_lp=25000),
                                      flg=P.flags(policy="FCFS")), "vllm")
        b = random_small_batch(rng, 3, 300)
        out = sim(cfg, b)
        check_invariants(b, out, cfg)
        for t in range(b.T):
            lo, hi = int(b.trace_off[t]), int(b.trace_off[t + 1])
            ins = inst(out["status"][lo:hi])
            assert list(ins) == [i % n_lp for i in range(hi - lo)]
            assert npre(out["status"][lo:hi]).sum() == 0
            ps = out["prefill_start_us"][lo:hi]
            for k in range(n_lp):
                q = ps[ins == k]
                assert np.all(np.diff(q) >= 0)


# ----------------------------------------------------- value functions and offload rules (f4) --
def w8_case(rule):
    g = H.golden("w8_lookahead_offload.json")
    t = g["topology"]
    cfg = H.tiny_cfg(n_lp=t["n_lp"], n_hp=t["n_hp"], block_tokens=t["block_tokens"],
                     kv_blocks=t["kv_blocks"], lp_max_batch=t["lp_max_batch"],
                     lp_token_budget=t["lp_token_budget"], hp_token_budget=t["hp_token_budget"],
                     policy="EDF_LAXITY", offload=1, tickets=0, elastic=0)
    cfg["flags"]["offload_rule"] = 0 if rule == "paper" else 1
    req = np.array(g["requests"], np.int64)
    b = TR.make_batch([(req[:, 0] * H.SEC, req[:, 1], req[:, 2])], [g["ttft"] * H.SEC], [g["tbt"] * H.SEC])
    return cfg, b, g["expect"][rule]


def check_w8(sim, goodput):
    for rule in ("paper", "lookahead"):
        cfg, b, exp = w8_case(rule)
        out = sim(cfg, b)
        assert [int(x) // H.SEC for x in out["first_token_us"]] == exp["first_token"], rule
        assert list((out["status"] >> 2) & 1) == exp["offloaded"], rule
        g, t = goodput(b, out)
        assert int(g[0]) == exp["good"], rule


WEIGHTED_EQUIV = [((1, -1, 0), "EDF_LAXITY"), ((1, 0, 0), "EDF_DEADLINE"), ((0, 1, 0), "SJF"),
                  ((0, -1, 0), "LJF"), ((0, 0, 1), "FCFS")]


def class_offsets(b, seed, premium_us=-2_000_000):
    """every other request (by a counter hash) is 'premium': its key moves premium_us earlier"""
    from gen.traces import mix_np
    h = mix_np(np.arange(b.R, dtype=np.uint64) + np.uint64(seed))
    return np.where((h & np.uint64(1)) == 1, premium_us, 0).astype(np.int64)
