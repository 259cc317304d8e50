mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -s -k "culling or render or raycast" -p no:cacheprovider > gpurun_out/pytest_render.log 2>&1; echo pytest=$?
timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c5.log 2>&1; echo bench=$?
