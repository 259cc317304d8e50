# compute-sanitizer over one small case of every kernel family (scripts/sanitize_cases.py);
# only this library's kernels are checked (mangled names "<len>k_...").  Logs -> gpurun_out/sanitize_*.log
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
FILTER="--kernel-name regex=[0-9]k_[a-z]"
python scripts/sanitize_cases.py env grad query bindings > gpurun_out/sanitize_plain.log 2>&1; echo plain=$?
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra $FILTER --print-limit 50 python scripts/sanitize_cases.py env grad query bindings \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Invalid|Uninitialized" gpurun_out/sanitize_$tool.log | sort | uniq -c | head -8
done
