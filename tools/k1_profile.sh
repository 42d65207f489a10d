#!/bin/bash
# ncu --set full of one k1_tasks launch on the row-S shape (GPU box; outputs under gpurun_out/<tag>*)
tag=${1:-k1}
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1_tasks -c 1 -o gpurun_out/${tag} \
  python tools/profile_run.py step --S ${S:-4096} --Q ${Q:-10000} --reps 2 > gpurun_out/${tag}.log 2>&1
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_src.csv
ncu -i gpurun_out/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv
tail -2 gpurun_out/${tag}.log
