"""Runs of equal execution count in an ncu SASS source export (--page source --csv --print-source sass):
where a kernel's executed instructions go.  usage: ncu_runs.py src.csv [min_share] [listing_start_suffix listing_end_suffix]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows[:5]) if 'Address' in r)
h = rows[hi]; data = rows[hi + 1:]
ia, isrc, iex = h.index('Address'), h.index('Source'), h.index('Instructions Executed')
iss = h.index('Warp Stall Sampling (All Samples)')
tot = sum(int(d[iex] or 0) for d in data)
smp = sum(int(d[iss] or 0) for d in data)
print('executed', tot, 'stall samples', smp)
if len(sys.argv) > 3:
    on = False
    for d in data:
        if d[ia].endswith(sys.argv[3]): on = True
        if on:
            print(d[ia][-5:], f"{int(d[iex] or 0):9d} {int(d[iss] or 0):6d}", d[isrc][:100])
            if d[ia].endswith(sys.argv[4]): break
    sys.exit()
ms = float(sys.argv[2]) if len(sys.argv) > 2 else 0.005
acc = []; prev = None; start = None; n = 0; s = 0
for d in data:
    e = int(d[iex] or 0)
    if e != prev:
        if prev: acc.append((start, n, prev, s))
        prev, start, n, s = e, d[ia], 0, 0
    n += 1; s += int(d[iss] or 0)
acc.append((start, n, prev, s))
for a, n, e, s in acc:
    if e and n * e > tot * ms:
        print(a[-6:], f"{n:5d} x {e:9d} = {n*e/tot*100:5.1f}% inst, {s/smp*100:5.1f}% stalls")
