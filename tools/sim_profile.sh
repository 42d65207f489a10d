#!/bin/bash
# ncu --set full of one sim_kernel launch (config-3 grid, shortened traces; GPU box)
tag=${1:-sim}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sim_kernel -c 1 -o gpurun_out/${tag} \
  python tools/profile_run.py sim --traces ${T:-4096} --n ${N:-1000} --reps 1 > gpurun_out/${tag}.log 2>&1
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_src.csv
ncu -i gpurun_out/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv
tail -2 gpurun_out/${tag}.log
