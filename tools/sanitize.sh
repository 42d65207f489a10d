# compute-sanitizer over every kernel family (tools/sanitize_run.py): memcheck, racecheck, synccheck,
# initcheck; logs to gpurun_out/<tag>_san_<tool>.log.  GPU box only.
tag=${1:-r02}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  # (no leak check: the torch caching allocator keeps its blocks until exit)
  timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 99 --print-limit 50 \
    python tools/sanitize_run.py > gpurun_out/${tag}_san_${tool}.log 2>&1
  echo "$tool rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY|sanitize_run done" gpurun_out/${tag}_san_${tool}.log | tail -3
done
