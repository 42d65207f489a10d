#!/bin/bash
# SASS bytes per device function of a csrc/*.cu file (I-cache budget check)
set -e
f=${1:-sim}
nvcc -cubin -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false ${EXTRA} \
  -o /tmp/$f.cubin paper_2504_20828_b200/csrc/$f.cu
readelf -sW /tmp/$f.cubin 2>/dev/null | python3 -c '
import sys, re
rows = []
for l in sys.stdin:
    p = l.split()
    if len(p) >= 8 and p[3] == "FUNC":
        sz = int(p[2], 0)
        nm = p[7]
        m = re.findall(r"\d+([a-z_][a-z_0-9]*?)E(?:RK|v|N)", nm)
        rows.append((sz, m[-1] if m else nm[-50:]))
for sz, nm in sorted(rows):
    print(f"{sz:8d} {nm}")
print(f"{sum(s for s, _ in rows):8d} total")
'
