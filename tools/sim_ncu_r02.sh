# sim_kernel captures on the bench's config-3 launch (calibrated preset): single-pass DRAM/instruction
# metrics of the full launch, then ncu --set full with source; GPU box only
tag=${1:-r02}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_bytes.sum,l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum,l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum \
  --clock-control none -k regex:sim_kernel -c 1 --csv --log-file gpurun_out/${tag}_sim_metrics.csv \
  python tools/profile_run.py sim --traces 4096 --n 10000 --reps 1 > gpurun_out/${tag}_sim_metrics.log 2>&1
echo metrics_rc=$?
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:sim_kernel -c 1 -o gpurun_out/${tag}_sim_full \
  python tools/profile_run.py sim --traces 4096 --n 10000 --reps 1 > gpurun_out/${tag}_sim_full.log 2>&1
echo full_rc=$?
ncu -i gpurun_out/${tag}_sim_full.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sim_src.csv
ncu -i gpurun_out/${tag}_sim_full.ncu-rep --page raw --csv > gpurun_out/${tag}_sim_raw.csv
