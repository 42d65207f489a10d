"""Markdown summary of a one-kernel ncu --set full raw CSV export (key counters + stall reasons).
usage: ncu_summary.py raw.csv title [command]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h, u, v = rows[0], rows[1], rows[2]
get = lambda k: (v[h.index(k)], u[h.index(k)]) if k in h else (None, None)
print(f"# {sys.argv[2]}\n")
if len(sys.argv) > 3:
    print(f"Command: `{sys.argv[3]}` (serialised replay; not a bench number)\n")
print(f"- Kernel: {get('Kernel Name')[0]} (grid {get('launch__grid_size')[0]} x block {get('launch__block_size')[0]}, "
      f"{get('launch__registers_per_thread')[0]} registers)")
for k, lab in (("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
               ("dram__bytes_write.sum", "DRAM write"), ("smsp__inst_executed.sum", "warp-instructions"),
               ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active"),
               ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active"),
               ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput"),
               ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts"),
               ("lts__t_bytes.sum", "L2 bytes")):
    val, unit = get(k)
    if val is not None:
        print(f"- {lab} (`{k}`): {val} {unit}")
print("- stalls (cycles per issued instruction): " + ", ".join(
    f"{n[34:-23]} {float(v[i]):.2f}" for i, n in enumerate(h)
    if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")
    and v[i] not in ("", "n/a") and float(v[i]) >= 0.1))
