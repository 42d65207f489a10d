# round-2 GPU session driver: bash tools/gpu_r02.sh <tag> <step>...
tag=$1; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for w in "$@"; do
  case $w in
    tests) timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -5 gpurun_out/${tag}_pytest_gpu.log;;
    testsfast) timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -5 gpurun_out/${tag}_pytest_gpu.log;;
    bench) timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/${tag}_bench.log 2> gpurun_out/${tag}_bench.err; echo bench_rc=$?; tail -c 4000 gpurun_out/${tag}_bench.log; tail -5 gpurun_out/${tag}_bench.err;;
    smoke) timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo smoke_rc=$?; tail -3 gpurun_out/${tag}_smoke.log;;
    *) echo "running: $w"; timeout 1800 bash -c "$w"; echo "rc=$?";;
  esac
done
