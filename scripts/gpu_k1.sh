# K1 variants: register caps (dynamics roofline)
mkdir -p gpurun_out
for m in 6 5 4; do
  python -m paper_2407_14783_b200.build -D QB_DYN_MINB=$m > /dev/null 2>&1
  timeout 600 python bench.py --workload c1 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/k1_$m.log 2>&1; echo k1_$m=$?
done
python -m paper_2407_14783_b200.build --force > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_gradients.py tests/test_gpu_env.py -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
