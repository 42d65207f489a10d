#!/bin/bash
# One gpurun call's worth of evidence at HEAD (GPU box only): bash tools/gpu_call.sh <tag> [steps...]
# steps: smoke tests bench launches traffic simfull ksfull k1full sanitize  (default: all but sanitize)
tag=$1; shift
[ $# -eq 0 ] && set -- smoke tests bench launches traffic simfull
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum"
ML="$M,l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum,l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum"
cap() { # name kernel-regex count args...
  local name=$1 k=$2 c=$3; shift 3
  timeout 1200 ncu --metrics $ML --clock-control none -k regex:$k -c $c --csv \
    --log-file gpurun_out/${tag}_${name}_dram.csv python tools/profile_run.py "$@" > gpurun_out/${tag}_${name}_dram.log 2>&1
  echo "cap $name rc=$?"
}
for s in "$@"; do
  t0=$(date +%s)
  case $s in
    smoke) timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
           echo smoke_rc=$?; tail -3 gpurun_out/${tag}_smoke.log;;
    tests) timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/${tag}_pytest_gpu.log 2>&1
           echo pytest_rc=$?; tail -22 gpurun_out/${tag}_pytest_gpu.log;;
    testsfast) timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1
           echo pytest_rc=$?; tail -5 gpurun_out/${tag}_pytest_gpu.log;;
    bench) timeout 1500 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
           echo bench_rc=$?; tail -c 6000 gpurun_out/${tag}_bench.json; tail -5 gpurun_out/${tag}_bench.err;;
    benchref) timeout 900 python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2>&1; echo ref_rc=$?
           cat gpurun_out/${tag}_bench_ref.json | tail -c 1500;;
    launches) timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
           --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
           --no-baselines > gpurun_out/${tag}_launches_bench.log 2>&1; echo launches_rc=$?;;
    traffic)
      cap sim sim_kernel 1 sim --traces 4096 --n 10000 --reps 1
      cap sim_config4 sim_kernel 1 sim --workload config4 --traces 1 --n 1000000 --reps 1
      cap k1 k1_tasks 2 step --S 4096 --Q 10000 --reps 2
      cap klane k_lane 2 step --S 1000000 --Q 32 --reps 2
      cap fit fit_partials 2 fit --reps 2
      python tools/ncu_traffic.py gpurun_out/${tag}_ncu_traffic.json \
        sim_kernel=gpurun_out/${tag}_sim_dram.csv sim_kernel_config4=gpurun_out/${tag}_sim_config4_dram.csv \
        k1_tasks=gpurun_out/${tag}_k1_dram.csv k_lane=gpurun_out/${tag}_klane_dram.csv \
        fit_partials=gpurun_out/${tag}_fit_dram.csv
      cp gpurun_out/${tag}_ncu_traffic.json profiles/ncu_traffic_r02.json;;  # read by the bench step after it
    simfull) timeout 2400 ncu --set full --import-source on --clock-control none -k regex:sim_kernel -c 1 \
           -o gpurun_out/${tag}_sim_full python tools/profile_run.py sim --traces 4096 --n 10000 --reps 1 \
           > gpurun_out/${tag}_sim_full.log 2>&1; echo simfull_rc=$?
           ncu -i gpurun_out/${tag}_sim_full.ncu-rep --page raw --csv > gpurun_out/${tag}_sim_raw.csv
           ncu -i gpurun_out/${tag}_sim_full.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sim_src.csv;;
    ksfull) bash tools/ks_profile.sh ${tag}_ks;;
    k1full) timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1_tasks -c 1 \
           -o gpurun_out/${tag}_k1_full python tools/profile_run.py step --S 4096 --Q 10000 --reps 2 \
           > gpurun_out/${tag}_k1_full.log 2>&1; echo k1full_rc=$?
           ncu -i gpurun_out/${tag}_k1_full.ncu-rep --page raw --csv > gpurun_out/${tag}_k1_raw.csv
           ncu -i gpurun_out/${tag}_k1_full.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_k1_src.csv;;
    sanitize) bash tools/sanitize.sh $tag;;
    steptests) timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_edges.py -x -q > gpurun_out/${tag}_steptests.log 2>&1
           echo steptests_rc=$?; tail -15 gpurun_out/${tag}_steptests.log;;
    timestep) timeout 600 python tools/time_step.py 2>&1 | tee gpurun_out/${tag}_timestep.log;;
    klanefull) timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_lane -c 1 \
           -o gpurun_out/${tag}_kl python tools/profile_run.py step --S 1000000 --Q 32 --reps 2 > gpurun_out/${tag}_kl.log 2>&1
           echo klanefull_rc=$?
           ncu -i gpurun_out/${tag}_kl.ncu-rep --page raw --csv > gpurun_out/${tag}_kl_raw.csv
           ncu -i gpurun_out/${tag}_kl.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_kl_src.csv;;
    c4full) timeout 1800 ncu --set full --import-source on --clock-control none -k regex:sim_kernel -c 1 \
           -o gpurun_out/${tag}_c4 python tools/profile_run.py sim --workload config4 --traces 1 --n 100000 --reps 1 \
           > gpurun_out/${tag}_c4.log 2>&1; echo c4full_rc=$?
           ncu -i gpurun_out/${tag}_c4.ncu-rep --page raw --csv > gpurun_out/${tag}_c4_raw.csv
           ncu -i gpurun_out/${tag}_c4.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_c4_src.csv;;
    *) echo "running: $s"; timeout 1800 bash -c "$s"; echo "rc=$?";;
  esac
  echo "[$s took $(( $(date +%s) - t0 )) s]"
done
