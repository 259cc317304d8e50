# K2 culling kernel: parity + c3/c2 bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_env.py -q -x -p no:cacheprovider > gpurun_out/pytest_render.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_render.log
for w in c3 c2; do
timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/$w.log 2>&1; echo $w=$?
done
