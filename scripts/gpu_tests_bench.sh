mkdir -p gpurun_out
bash scripts/gpu_tests.sh
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench=$?
tail -2 gpurun_out/bench.log
