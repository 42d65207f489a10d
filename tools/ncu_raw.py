"""Key counters of a one-kernel ncu raw CSV export: time, DRAM bytes, instructions, issue, stalls."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h, u, v = rows[0], rows[1], rows[2]
want = ['gpu__time_duration.sum', 'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__cycles_active.avg', 'gpc__cycles_elapsed.max', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__t_bytes.sum', 'l1tex__t_bytes.sum']
for i, n in enumerate(h):
    if n in want:
        print(f"{n:60s} {v[i]:>16s} {u[i]}")
for i, n in enumerate(h):
    if n.startswith('smsp__average_warps_issue_stalled_') and n.endswith('_per_issue_active.ratio'):
        try:
            if float(v[i]) > 0.1:
                print(f"  {n[34:-23]:40s} {float(v[i]):.2f}")
        except ValueError:
            pass
