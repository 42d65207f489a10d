#!/bin/bash
# ncu --set full of one k_small launch on the row-S short-queue shape (10^6 segments x 32; GPU box)
tag=${1:-ks}
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_small -c 1 -o gpurun_out/${tag} \
  python tools/profile_run.py step --S 1000000 --Q 32 --reps 2 > gpurun_out/${tag}.log 2>&1
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_src.csv
ncu -i gpurun_out/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv
tail -2 gpurun_out/${tag}.log
