mkdir -p gpurun_out
bash scripts/gpu_tests.sh
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c3.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_c3.log | cut -c1-200
