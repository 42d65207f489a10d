#!/bin/bash
# Run on the GPU box (via gpurun): bench line, ncu launch list of the bench command, and the
# single-pass DRAM traffic of the two roofline kernels.  Outputs land in gpurun_out/<tag>_*.
# Numbers printed under ncu are never bench values; the bench line comes from the plain run.
tag=${1:-r01}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
tail -c 3000 gpurun_out/${tag}_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-baselines --no-fit-bench \
  > gpurun_out/${tag}_launches_bench.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum \
  --clock-control none -k regex:sim_kernel -c 1 --csv --log-file gpurun_out/${tag}_sim_dram.csv \
  python tools/profile_run.py sim --traces 4096 --n 10000 --reps 1 > gpurun_out/${tag}_sim_dram.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:k1_tasks -c 2 --csv --log-file gpurun_out/${tag}_k1_dram.csv \
  python tools/profile_run.py step --S 4096 --Q 10000 --reps 2 > gpurun_out/${tag}_k1_dram.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:fit_partials -c 2 --csv --log-file gpurun_out/${tag}_fit_dram.csv \
  python tools/profile_run.py fit --reps 2 > gpurun_out/${tag}_fit_dram.log 2>&1
echo done
