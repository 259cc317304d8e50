# split env step: parity + A/B on the small-batch camera workloads
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_split.py -q -rf --tb=short -p no:cacheprovider > gpurun_out/pytest_split.log 2>&1; echo split_pytest=$?
tail -15 gpurun_out/pytest_split.log
for r in 1 2; do for sp in 0 1; do for w in c2 c2a; do
  QB_SPLIT_STEP=$sp timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/sp_${sp}_$w.log 2>&1
  echo "split=$sp $w $(tail -1 gpurun_out/sp_${sp}_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])" 2>&1 | tail -1)"
done; done; done
bash scripts/gpu_tests.sh
