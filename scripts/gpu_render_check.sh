mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -s -k "culling or render" -p no:cacheprovider > gpurun_out/pytest_render.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c3.log 2>&1; echo bench=$?
