# parity suite + C3 bench + swarm and c2a lines (culling renderer changes)
mkdir -p gpurun_out
bash scripts/gpu_tests.sh
for w in ${WL:-c3 c2a swarm}; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$w.log 2>&1; echo $w=$?
  tail -1 gpurun_out/bench_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('kernel_ms'))"
done
