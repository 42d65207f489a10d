#!/usr/bin/env python
"""bench.py — scheduler decisions/s and simulated requests/s of the sm_100a hot path.

One "step" = one pass of the whole hot path over one batch of synthetic input: asc_simulate_batch
(rows a1-a7: perf model, keys, Algorithm 1 selection, offload/drop compaction, batch latency,
event loop) followed by asc_goodput (row a8) on BASELINE.json config 3: 4096 independent traces
(16 QPS x 16 SLO scales x 16 seeds) x 10k ShareGPT-shaped requests, 2 LP + 1 HP, Mistral-7B /
A100 perf model.  With --gpus N (torchrun, one rank per GPU) every rank simulates its own
config-3 grid with seed 1 + rank (weak scaling; traces never interact, so there is no data-path
collective); integer goodput counters are all-reduced over NCCL once at the end.

Also reported on the same line: the HBM roofline of the dominant kernel, the stateless
asc_schedule_step microbenchmark with its own roofline, the CPU oracle on a
bounded sample (cpu_baseline), and an end-to-end number through the C ABI with host buffers.
`--impl reference` times the CPU oracle instead (the reference arm for this tier).
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from gen import presets as P  # noqa: E402

METRIC = "scheduler decisions/sec"
UNIT = "decisions/s"
FALLBACK_HBM = 6650.0


def args_():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="asc", choices=["asc", "reference"])
    ap.add_argument("--workload", default="config3")
    ap.add_argument("--no-baselines", action="store_true", help="skip the baseline scheduler runs")
    ap.add_argument("--no-fit-bench", action="store_true", help="skip the perf-model fit microbench")
    ap.add_argument("--requests", type=int, default=None, help="requests per trace override")
    ap.add_argument("--traces", type=int, default=None, help="max traces (testing)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-step-bench", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-config4", action="store_true", help="skip the BASELINE config 4 sub-line")
    ap.add_argument("--no-config5", action="store_true", help="skip the BASELINE config 5 shard sub-line")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM, "fallback (B200_PROFILING.md 6.65 TB/s)"


NCU_TRAFFIC = os.path.join(ROOT, "profiles", "ncu_traffic_r02.json")


def ncu_traffic(kernel):
    """{"bytes": dram read+write bytes per launch, "inst": warp-instructions per launch (optional),
    "source": capture} from one ncu capture of the same launch configuration at this round's code
    (profiles/ncu_traffic_r02.json, written by tools/ncu_traffic.py), or None."""
    if os.path.exists(NCU_TRAFFIC):
        with open(NCU_TRAFFIC) as f:
            v = json.load(f).get(kernel)
        return v if isinstance(v, dict) else None
    return None


def traffic_bytes(kernel):
    v = ncu_traffic(kernel)
    return v.get("bytes") if v else None


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(", ") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[0]) for r in rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        if not sm:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 7 for i in range(4)
                          if r[3 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(sm)}


def load(name, rank, world, n, traces):
    """-> (cfg, batch, desc, point_of_trace, grid) where grid describes the (QPS, SLO-scale) points."""
    if name == "config3":
        cfg, b = P.workload("config3", n=n, max_traces=traces, base_seed=1 + rank)
        desc = f"config3 (4096 traces x 10k ShareGPT-shaped req, 2L1H, calibrated perf preset, seed {1 + rank}"
        desc += ")" if world == 1 else f", one grid per rank: {world} x 4096 traces)"
        grid = dict(n_qps=16, n_scale=16, qps=[(q + 1) / 2 for q in range(16)],
                    scale=[(k + 1) / 4 for k in range(16)], scale1=3)
    elif name == "config5":   # 65536 traces x 100k sharded i = rank mod world
        cfg, full = P.workload("config5", n=1, max_traces=traces)
        idx = list(range(rank, full.T, world))   # only this rank's grid points are generated
        cfg, b = P.workload("config5", n=n or 100_000, max_traces=traces, select=idx)
        desc = f"config5 shard {rank}/{world} (calibrated perf preset)"
        grid = dict(n_qps=64, n_scale=64, qps=[(q + 1) / 8 for q in range(64)],
                    scale=[(k + 1) / 16 for k in range(64)], scale1=15)
    elif name in ("config1", "config2", "config4"):
        cfg, b = P.workload(name, n=n, max_traces=traces, base_seed=1 + rank)
        desc = f"{name} ({P.DEFAULT_PERF[name]} perf preset)"
        grid = None
    else:
        raise SystemExit(f"unknown workload {name}")
    tidx = np.array([int(l.split(":")[0][1:]) for l in b.labels], np.int64)
    point = tidx // 16 if grid else tidx
    return cfg, b, desc, point, grid


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_baseline(cfg, batch, budget_s=12.0):
    """The oracle as it stands, on a stratified sample of traces, all host cores.  A probe of
    2 x cores traces sizes the measured sample to about budget_s seconds of CPU work."""
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    T = batch.T

    def run(m):
        idx = sorted(set(np.linspace(0, T - 1, m).round().astype(int).tolist()))
        sub = batch.subset(idx)
        t0 = time.perf_counter()
        out = O.simulate_batch(cfg, sub, nthreads=cores)
        return idx, sub, out, time.perf_counter() - t0

    m = min(T, max(4, 2 * cores))
    idx, sub, out, dt = run(m)
    if dt < 0.5 * budget_s and m < T:
        idx, sub, out, dt = run(min(T, int(m * budget_s / max(dt, 1e-3))))
    dec = int(out["decisions"].sum())
    return {"value": dec / dt, "unit": UNIT, "cores": min(cores, len(idx)), "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"{len(idx)} of {T} traces (stratified over the QPS x SLO grid), "
                      f"{sub.R} requests, {dec} decisions in {dt:.2f} s",
            "simulated_req_per_s": sub.R / dt,
            "evaluations_per_s": int(out["evaluations"].sum()) / dt, "seconds": dt}


def reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg, b, desc, _, _ = load(a.workload, 0, 1, a.requests, a.traces)
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    per_step = min(b.T, max(4, cores))
    vals, reqs, secs = [], [], []
    rng = np.random.default_rng(0)
    # each step is a bounded random sample; the first warm-up step sizes it to ~target_s seconds
    target_s = max(1.0, min(6.0, 150.0 / max(1, a.warmup + a.steps)))
    for step in range(a.warmup + a.steps):
        idx = sorted(rng.choice(b.T, size=per_step, replace=False).tolist())
        sub = b.subset(idx)
        t0 = time.perf_counter()
        out = O.simulate_batch(cfg, sub, nthreads=cores)
        dt = time.perf_counter() - t0
        if step == 0:
            per_step = int(min(b.T, max(per_step, per_step * target_s / max(dt, 1e-3))))
        if step >= a.warmup:
            vals.append(int(out["decisions"].sum()))
            reqs.append(sub.R)
            secs.append(dt)
    v = sum(vals) / sum(secs)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1000 * sum(secs) / len(secs),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64/f64",
            "data": "synthetic",
            "config": {"workload": desc, "sample_traces_per_step": per_step},
            "simulated_req_per_s": sum(reqs) / sum(secs),
            "cpu_baseline": {"value": v, "unit": UNIT, "kind": "oracle", "cores": min(cores, per_step),
                             "cpu_model": cpu_model(),
                             "sample": f"{per_step} random traces of {b.T} per step"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def step_microbench(asc, torch, dev, stream, warmup, steps, hbm_peak):
    """Row S: asc_schedule_step on 4096 segments x 10,000 entries (ShareGPT prompt mix, deadlines
    now +- 3 s, random budgets), the deep-queue shape of SURVEY §8(d)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import helpers as H
    rng = np.random.default_rng(123)
    cfg = P.config()
    S, Qs = 4096, 10_000
    ins = H.random_step_inputs(rng, S, 0, cfg, qs=np.full(S, Qs))
    dins = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in ins.items()}
    dins["Q"] = S * Qs
    ctx = asc.Context(cfg, dev.index, stream)
    Q = S * Qs
    out = None
    for _ in range(warmup):
        out = ctx.schedule_step(dins, want_prefill=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    k1 = []
    e0.record(stream)
    for _ in range(steps):
        out = ctx.schedule_step(dins, want_prefill=False, out=out)
        k1.append(ctx.last_kernel_ms())
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    nout = int(out["admit_cnt"].sum() + out["offload_cnt"].sum() + out["drop_cnt"].sum())
    # 12 B per request evaluation (deadline 8 B + eff_prompt 4 B with the flag bits
    # packed in); the ABI's separate flag byte (13 B moved per entry) is not credited
    byts = 12 * Q + 4 * nout + S * (8 * 4 + 4 * 6) + 8
    k1ms = float(np.mean(k1))
    ctx.close()
    others = []
    for S2, Q2 in ((64, 1_000_000), (1_000_000, 32)):  # the other two row-S shapes
        ins2 = H.random_step_inputs(np.random.default_rng(123), S2, 0, cfg, qs=np.full(S2, Q2))
        d2 = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in ins2.items()}
        d2["Q"] = S2 * Q2
        c2 = asc.Context(cfg, dev.index, stream)
        for _ in range(warmup):
            o2 = c2.schedule_step(d2, want_prefill=False)
        torch.cuda.synchronize()
        kl = []
        e0.record(stream)
        for _ in range(steps):
            o2 = c2.schedule_step(d2, want_prefill=False, out=o2)
            kl.append(c2.last_kernel2_ms())
        e1.record(stream)
        torch.cuda.synchronize()
        ms2 = e0.elapsed_time(e1) / steps
        n2 = int(o2["admit_cnt"].sum() + o2["offload_cnt"].sum() + o2["drop_cnt"].sum())
        b2 = 12 * S2 * Q2 + 4 * n2 + S2 * (8 * 4 + 4 * 6) + 8
        c2.close()
        sh = {"shape": f"S={S2} segments x Q={Q2} entries", "ms_per_call": ms2,
              "evaluations_per_s": S2 * Q2 / (ms2 * 1e-3),
              "whole_call_achieved_gbs": b2 / (ms2 * 1e-3) / 1e9,
              "whole_call_frac": b2 / (ms2 * 1e-3) / 1e9 / hbm_peak}
        if Q2 <= 32:  # every segment is k_lane's (one thread per segment)
            klm = float(np.mean(kl))
            sh["roofline"] = {"bound": "hbm", "kernel": "k_lane (one thread per short segment)",
                              "achieved": b2 / (klm * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                              "frac": b2 / (klm * 1e-3) / 1e9 / hbm_peak, "kernel_ms": klm,
                              "algorithmic_bytes": b2, "traffic": traffic_bytes("k_lane")}
        others.append(sh)
        del d2, o2
    ach_k1 = byts / (k1ms * 1e-3) / 1e9     # single-task segments: k1 does all reads and writes
    ach_call = byts / (ms * 1e-3) / 1e9
    return {"shape": f"S={S} segments x Q={Qs} entries", "entries": Q,
            "ms_per_call": ms, "evaluations_per_s": Q / (ms * 1e-3),
            "admitted": int(out["admit_cnt"].sum()), "offloaded": int(out["offload_cnt"].sum()),
            "roofline": {"bound": "hbm", "achieved": ach_k1, "peak": hbm_peak, "unit": "GB/s",
                         "frac": ach_k1 / hbm_peak, "traffic": traffic_bytes("k1_tasks"),
                         "kernel": "k1_tasks (streaming pass; finishes every single-task segment)",
                         "algorithmic_bytes": byts, "kernel_ms": k1ms, "kernel_share": k1ms / ms},
            "whole_call": {"achieved": ach_call, "unit": "GB/s", "frac": ach_call / hbm_peak,
                           "note": "asc_schedule_step incl. planner launch and the error sync"},
            "other_shapes": others}


def maybe_spawn(a):
    """`bench.py --gpus N` without torchrun: re-launch under torch.distributed.run with N ranks."""
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1", "--master-port",
               str(port), os.path.abspath(__file__)] + sys.argv[1:]
        os.execv(sys.executable, cmd)


def grid_report(grid, tab, rows_all, point_all):
    """Per-grid-point table (all ranks) -> the goodput surface and the SLO-scale-1 row."""
    from paper_2504_20828_b200 import dist as D
    col = {k: tab[:, j].astype(np.float64) for j, k in enumerate(D.POINT_COUNTERS)}
    nq, ns = grid["n_qps"], grid["n_scale"]
    div = lambda x, y: np.where(y > 0, x / np.maximum(y, 1), np.nan)
    gp = div(col["good"], col["total"]).reshape(nq, ns)
    s1 = grid["scale1"]
    at = lambda v: [None if not np.isfinite(x) else round(float(x), 4) for x in v.reshape(nq, ns)[:, s1]]
    # p99 TTFT per point: median over the point's traces of the per-trace nearest-rank p99
    p99 = np.full(nq * ns, np.nan)
    for pnt in np.unique(point_all):
        v = rows_all[point_all == pnt, 1]
        v = v[v >= 0]
        if len(v):
            p99[pnt] = np.median(v) / 1e3
    ev_req = div(col["evaluations"], col["total"])
    batch = div(col["tokens"], col["decisions"])
    over = slice(nq // 2, nq)
    return {
        "qps": grid["qps"], "slo_scale": grid["scale"],
        "goodput_surface": [[None if not np.isfinite(x) else round(float(x), 3) for x in r] for r in gp]
        if nq * ns <= 256 else "omitted (see at_slo_scale_1)",
        "at_slo_scale_1": {
            "goodput": at(div(col["good"], col["total"])),
            "evaluations_per_request": at(ev_req), "decisions_per_request": at(div(col["decisions"], col["total"])),
            "mean_batch_requests": at(batch), "p99_ttft_ms_median_over_seeds": at(p99),
            "mean_tbt_ms": at(div(col["tbt_sum_us"], col["tbt_tokens"]) / 1e3),
            "sched_delay_lp_ms": at(div(col["delay_sum_lp_us"], col["delay_cnt_lp"]) / 1e3),
            "sched_delay_hp_ms": at(div(col["delay_sum_hp_us"], col["delay_cnt_hp"]) / 1e3),
            "dropped_frac": at(div(col["dropped"], col["total"]))},
        "overloaded_half_at_scale_1": {
            "qps": grid["qps"][nq // 2:],
            "evaluations_per_request": round(float(np.nansum(col["evaluations"].reshape(nq, ns)[over, s1])
                                                   / np.nansum(col["total"].reshape(nq, ns)[over, s1])), 2),
            "mean_batch_requests": round(float(np.nansum(col["tokens"].reshape(nq, ns)[over, s1])
                                               / np.nansum(col["decisions"].reshape(nq, ns)[over, s1])), 2)},
        "mean_batch_requests_all": round(float(col["tokens"].sum() / max(col["decisions"].sum(), 1)), 2),
        "evaluations_per_request_all": round(float(col["evaluations"].sum() / max(col["total"].sum(), 1)), 2),
        "note": "mean batch = generated tokens / non-empty formations (every batch member emits one token)",
    }


def main():
    a = args_()
    maybe_spawn(a)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}")
    if a.impl == "reference":
        return reference_arm(a)
    import torch
    from paper_2504_20828_b200 import asc
    from paper_2504_20828_b200 import dist as D
    assert torch.cuda.is_available(), "bench.py needs CUDA (no CPU fallback)"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    hbm_peak, peak_src = peaks()
    cfg, batch, desc, point, grid = load(a.workload, rank, world, a.requests, a.traces)
    stream = torch.cuda.Stream(device=dev)
    ctx = asc.Context(cfg, local, stream)
    tr = asc.batch_arrays(batch, dev)
    out = ctx.simulate_batch(tr)
    res = {k: torch.empty(max(batch.T, 1), dtype=torch.int64, device=dev) for k in ("good", "total")}
    summ = {k: torch.empty(max(batch.T, 1), dtype=torch.int64, device=dev) for k in asc.SUMMARY_KEYS}
    ctx.goodput(tr, out, res=res)
    ctx.summarize(tr, out, res=summ)

    def step():
        # one pass of the hot path: simulate (rows a1-a7) + goodput and outcome summary (row a8)
        ctx.simulate_batch(tr, out=out)
        sim_ms = ctx.last_kernel_ms()
        l1 = ctx.last_launches()
        ctx.goodput(tr, out, res=res)
        l2 = ctx.last_launches()
        ctx.summarize(tr, out, res=summ)
        return sim_ms, l1 + l2 + ctx.last_launches()

    for _ in range(max(0, a.warmup - 1)):
        step()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    barrier()
    torch.cuda.synchronize()
    clk = Clocks(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    sims, launches = [], 0
    for _ in range(a.steps):
        ms, l = step()
        sims.append(ms)
        launches += l
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    ms_total = e0.elapsed_time(e1)
    T = batch.T
    host = lambda x: x[:T].cpu().numpy()
    per_trace = {k: host(summ[k]) for k in asc.SUMMARY_KEYS}
    per_trace.update(good=host(res["good"]), total=host(res["total"]), decisions=host(out["decisions"]),
                     evaluations=host(out["evaluations"]),
                     finished=per_trace["completed"] + per_trace["dropped"])
    n_points = (grid["n_qps"] * grid["n_scale"]) if grid else int(point.max()) + 1
    tab = D.reduce_points(D.point_counters(point, n_points, per_trace), dev)
    rows = np.stack([host(out["digest"]), per_trace["ttft_p99_us"], point], 1)
    parts = D.gather_rows(rows, dev)
    rows_all = np.concatenate(parts, 0)
    col = {k: int(tab[:, j].sum()) for j, k in enumerate(D.POINT_COUNTERS)}
    dec_all, evals_all, fin_all = col["decisions"], col["evaluations"], col["finished"]
    ms_step = D.reduce_max(ms_total, dev) / a.steps
    value = dec_all / (ms_step * 1e-3)
    sim_ms = float(np.mean(sims))
    evals = int(per_trace["evaluations"].sum())
    algo = 44 * batch.R + 12 * evals          # SURVEY §8(d)'s figure, this rank
    ach = algo / (sim_ms * 1e-3) / 1e9
    traffic = ncu_traffic("sim_kernel") if a.workload == "config3" else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64/f64", "data": "synthetic",
        "config": {"workload": desc, "traces_per_gpu": batch.T, "requests_per_gpu": batch.R,
                   "parallelism": f"dp{world} (independent traces, no data-path collective)",
                   "l2": "inputs+workspace > 126 MB L2 (no flush needed)",
                   "perf_model": "Mistral-7B shape, A100 caps 312 TF / 2 TB/s, C=" + str(tuple(cfg["perf"]["c"]))},
        "simulated_req_per_s": fin_all / (ms_step * 1e-3),
        "evaluations_per_s": evals_all / (ms_step * 1e-3),
        "goodput": col["good"] / max(col["total"], 1),
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                     "frac": ach / hbm_peak, "traffic": traffic.get("bytes") if traffic else None,
                     "kernel": "sim_kernel (event loop)", "peak_source": peak_src,
                     "note": "algorithmic bytes = SURVEY 8(d)'s 44 B per request + 12 B per queued-request "
                             "evaluation; the sorted-queue kernel touches O(admitted + offloaded) entries per "
                             "formation, not every queued one, so this credits reads it does not make (an "
                             "upper bound); traffic = ncu dram bytes of one launch (profiles/ncu_traffic_r02.json). "
                             "The event loop is a dependent chain per trace: issue-bound, see issue_roofline",
                     "algorithmic_bytes": algo, "kernel_ms": sim_ms,
                     "kernel_share": sim_ms / ms_step},
        "clocks": clocks,
    }
    if grid:
        line["grid"] = grid_report(grid, tab, rows_all, rows_all[:, 2])
    if traffic:
        line["roofline"]["traffic_source"] = traffic.get("source")
        inst = traffic.get("inst")
        if inst:
            sms = torch.cuda.get_device_properties(dev).multi_processor_count
            mhz = (clocks or {}).get("sm_max_mhz") or 1965.0
            ipk = 4 * sms * mhz * 1e6          # 4 schedulers per SM, 1 warp-instruction per cycle each
            ach_i = inst / (sim_ms * 1e-3)
            line["issue_roofline"] = {"bound": "issue", "achieved": ach_i, "peak": ipk, "unit": "warp-inst/s",
                                      "frac": ach_i / ipk, "inst_per_launch": inst,
                                      "source": traffic.get("source") + " (smsp__inst_executed.sum of one launch) "
                                                "over the live kernel time; peak = 4 schedulers x SMs x max SM clock"}
    if rank == 0 and not a.no_step_bench:
        line["step_microbench"] = step_microbench(asc, torch, dev, stream, 2, max(3, a.steps), hbm_peak)
    if not a.no_e2e:
        line["e2e"] = e2e(asc, torch, ctx, batch, world, max(3, a.steps), dev)
    if rank == 0 and not a.no_fit_bench:
        line["fit_microbench"] = fit_microbench(asc, torch, dev, stream, hbm_peak)
        line["latency_microbench"] = latency_microbench(asc, torch, dev, stream, hbm_peak)
    ctx.close()
    if rank == 0 and not a.no_baselines:
        line["baselines"] = baselines(asc, torch, dev, stream, cfg, batch, col["good"] / max(col["total"], 1))
    # configs 4 and 5 (one trace / one GPU's shard) are single-GPU lines: the N = 1 run carries them
    if rank == 0 and world == 1 and not a.no_config4:
        line["config4"] = config4_line(asc, torch, dev, stream, hbm_peak)
    if rank == 0 and world == 1 and not a.no_config5:
        del tr, out, res, summ
        torch.cuda.empty_cache()
        line["config5_shard"] = config5_line(asc, torch, dev, stream)
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, batch)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def config4_line(asc, torch, dev, stream, hbm_peak):
    """BASELINE config 4 in full: one LongBench-shaped trace of 10^6 requests at QPS 12 (~2x the
    2L1H saturation), deep queues; one timed asc_simulate_batch + asc_goodput."""
    cfg, b = P.workload("config4")
    ctx = asc.Context(cfg, dev.index, stream)
    tr = asc.batch_arrays(b, dev)
    out = ctx.simulate_batch(tr)
    ms = ctx.last_kernel_ms()
    good, total = ctx.goodput(tr, out)
    dec = int(out["decisions"][:1].sum().item())
    ev = int(out["evaluations"][:1].sum().item())
    g = int(good[:1].cpu().numpy().view(np.uint64)[0])
    t = int(total[:1].cpu().numpy().view(np.uint64)[0])
    ctx.close()
    tr_ = traffic_bytes("sim_kernel_config4")
    return {"workload": "config4: 1 trace, 10^6 LongBench-shaped requests, 2L1H, QPS 12, roofline preset",
            "kernel_ms": ms, "decisions": dec, "evaluations": ev,
            "decisions_per_s": dec / (ms * 1e-3), "evaluations_per_s": ev / (ms * 1e-3),
            "simulated_req_per_s": b.R / (ms * 1e-3), "goodput": g / max(t, 1),
            "algorithmic_gbs": (44 * b.R + 12 * ev) / (ms * 1e-3) / 1e9,
            "dram_bytes": tr_,
            "note": "one trace = one warp's sequential event chain"}


def config5_line(asc, torch, dev, stream, W=16, r=0):
    """BASELINE config 5's per-GPU unit: shard r of W of the 65,536-trace x 100k-request QPS x SLO
    grid (traces i = r mod W, as dist.py shards it across ranks) = 4096 traces x 10^5 requests
    (4.1e8) on one B200; one timed asc_simulate_batch + asc_goodput after the uploads."""
    from paper_2504_20828_b200 import dist as D
    t0 = time.perf_counter()
    cfg, full = P.workload("config5", n=1)
    cfg, b = P.workload("config5", n=100_000, select=D.shard(full.T, r, W))
    gen_s = time.perf_counter() - t0
    ctx = asc.Context(cfg, dev.index, stream)
    tr = asc.batch_arrays(b, dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    out = ctx.simulate_batch(tr)
    sim_ms = ctx.last_kernel_ms()
    good, total = ctx.goodput(tr, out)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    dec = int(out["decisions"][:b.T].sum().item())
    ev = int(out["evaluations"][:b.T].sum().item())
    g = int(good[:b.T].cpu().numpy().view(np.uint64).sum())
    t = int(total[:b.T].cpu().numpy().view(np.uint64).sum())
    ctx.close()
    del tr, out, good, total
    torch.cuda.empty_cache()
    return {"workload": f"config5 shard {r}/{W}: {b.T} traces x 100k ShareGPT-shaped requests "
                        f"({b.R} requests), 2L1H, QPS 1/8..8 x SLO scale 1/16..4, calibrated preset",
            "ms": ms, "kernel_ms": sim_ms, "decisions": dec, "evaluations": ev,
            "decisions_per_s": dec / (ms * 1e-3), "simulated_req_per_s": b.R / (ms * 1e-3),
            "evaluations_per_s": ev / (ms * 1e-3), "goodput": g / max(t, 1), "host_gen_s": gen_s,
            "note": "one GPU's share of the 8-GPU config-5 grid (W = 16 shards; bench.py --gpus N "
                    "--workload config5 runs the grid sharded across N ranks)"}


def latency_microbench(asc, torch, dev, stream, hbm_peak, n=1 << 26, steps=5):
    """Rows a1/a6 alone: asc_latency over n device-resident (F, M) pairs (Eq. 4-5 + G17/G18, the
    evaluation every formation makes); 16 B read + 16 B written (lat_us, t_s) per pair."""
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    F = torch.floor(torch.pow(2.0, torch.rand(n, generator=g, device=dev, dtype=torch.float64) * 52)).to(torch.int64)
    M = torch.floor(torch.pow(2.0, torch.rand(n, generator=g, device=dev, dtype=torch.float64) * 52)).to(torch.int64)
    ctx = asc.Context(P.config(), dev.index, stream)
    lat = torch.empty(n, dtype=torch.int64, device=dev)
    ts = torch.empty(n, dtype=torch.float64, device=dev)
    for _ in range(2):
        asc.asc_latency(ctx.h, F, M, lat, ts, n=n)
    torch.cuda.synchronize()
    k_ms = []
    for _ in range(steps):
        asc.asc_latency(ctx.h, F, M, lat, ts, n=n)
        k_ms.append(ctx.last_kernel_ms())
    ctx.close()
    kms = float(np.mean(k_ms))
    byts = 32 * n
    ach = byts / (kms * 1e-3) / 1e9
    return {"shape": f"{n} (F, M) pairs", "evaluations_per_s": n / (kms * 1e-3),
            "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                         "frac": ach / hbm_peak, "traffic": None, "kernel": "latency_kernel (asc_latency)",
                         "algorithmic_bytes": byts, "kernel_ms": kms}}


def fit_microbench(asc, torch, dev, stream, hbm_peak, groups=1024, per=65536, steps=5):
    """Row f2: asc_fit_perf over groups x per synthetic batch records (gen/records.py), device
    resident; roofline on fit_partials (24 B per record: F, M, y) over its event-timed duration."""
    from gen import records as RC
    rec = RC.make_records(21, [per] * groups)
    N = int(rec["off"][-1])
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in rec.items()}
    d["N"] = N
    ctx = asc.Context(P.config(), dev.index, stream)
    for _ in range(2):
        ctx.fit_perf(d, 1e-8, errors=False)
    torch.cuda.synchronize()
    k_ms, launches = [], 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        ctx.fit_perf(d, 1e-8, errors=False)
        k_ms.append(ctx.last_kernel_ms())
        launches += ctx.last_launches()
    e1.record(stream)
    torch.cuda.synchronize()
    call_ms = e0.elapsed_time(e1) / steps
    coef, me, mx = ctx.fit_perf(d, 1e-8, errors=True)
    ctx.close()
    kms = float(np.mean(k_ms))
    byts = 24 * N
    ach = byts / (kms * 1e-3) / 1e9
    return {"shape": f"{groups} groups x {per} records", "records": N,
            "records_per_s": N / (call_ms * 1e-3), "ms_per_call": call_ms,
            "gpu_launches_per_call": launches / steps,
            "median_in_sample_rel_err": float(np.median(me.cpu().numpy())),
            "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                         "frac": ach / hbm_peak, "traffic": traffic_bytes("fit_partials"),
                         "kernel": "fit_partials (features + Gram partials, one HBM pass)",
                         "algorithmic_bytes": byts, "kernel_ms": kms, "kernel_share": kms / call_ms}}


def baselines(asc, torch, dev, stream, cfg, batch, ascendra_goodput):
    """Row f1: the same traces under the vLLM-like and Sarathi-like (chunk budget 512) baselines on
    the same number of homogeneous
    instances, one timed asc_simulate_batch after a warm-up; goodput beside Ascendra's."""
    res = {"ascendra_goodput": ascendra_goodput}
    for name in ("vllm", "sarathi"):
        c = {k: dict(v) for k, v in cfg.items()}
        c["topo"]["n_lp"] = cfg["topo"]["n_lp"] + cfg["topo"]["n_hp"]
        c["topo"]["n_hp"] = 0
        c["flags"].update(scheduler=P.SCHEDULER[name], offload=0, tickets=0)
        ctx = asc.Context(c, dev.index, stream)
        tr = asc.batch_arrays(batch, dev)
        out = ctx.simulate_batch(tr)
        out = ctx.simulate_batch(tr, out=out)
        ms = ctx.last_kernel_ms()
        good, total = ctx.goodput(tr, out)
        dec = int(out["decisions"][:batch.T].sum().item())
        g = int(good[:batch.T].cpu().numpy().view(np.uint64).sum())
        t = int(total[:batch.T].cpu().numpy().view(np.uint64).sum())
        ctx.close()
        res[name] = {"decisions_per_s": dec / (ms * 1e-3), "kernel_ms": ms, "goodput": g / max(t, 1),
                     "instances": f"{c['topo']['n_lp']} homogeneous (P:575)"}
    return res


def e2e(asc, torch, ctx, batch, world, steps, dev):
    """Same metric through the C ABI with pinned HOST buffers: each step uploads the traces,
    simulates, reads the outcomes back, then computes goodput (uploads outcomes, reads counters)."""
    def pinned(x):
        t = torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
        return t.numpy()
    tr = {k: (pinned(v) if k != "R" else v) for k, v in asc.batch_arrays(batch).items()}
    R, T = batch.R, batch.T
    out = {k: pinned(np.zeros(max(n, 1), dt)) for k, (n, dt) in dict(
        first_token_us=(R, np.int64), done_us=(R, np.int64), prefill_start_us=(R, np.int64),
        status=(R, np.uint32), digest=(T, np.uint64), decisions=(T, np.int64),
        evaluations=(T, np.int64)).items()}
    res = {k: pinned(np.zeros(max(T, 1), np.uint64)) for k in ("good", "total")}
    ctx.simulate_batch(tr, out=out)   # warm-up (staging buffers)
    ctx.goodput(tr, out, res=res)
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        ctx.simulate_batch(tr, out=out)
        ctx.goodput(tr, out, res=res)
    dt = (time.perf_counter() - t0) / steps
    tmax = torch.tensor([dt], dtype=torch.float64, device=dev)
    dec = torch.tensor([int(out["decisions"][:T].sum())], dtype=torch.int64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(tmax, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(dec)
    h2d = (8 * (T + 1) + 16 * R + 16 * T) + (8 * (T + 1) + 12 * R + 16 * T + 20 * R)
    d2h = (28 * R + 24 * T) + 16 * T
    return {"value": int(dec.item()) / float(tmax.item()), "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": steps,
            "timing": "host wall clock per step (calls are synchronous), max over ranks",
            "path": "asc_simulate_batch + asc_goodput with pinned host pointers (library stages H2D/D2H)"}


if __name__ == "__main__":
    main()
