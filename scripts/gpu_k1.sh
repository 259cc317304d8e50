# K1 variants: scalar vs env-pair kernel, register caps (dynamics roofline)
mkdir -p gpurun_out
for cfg in "0 8 3" "0 6 3" "1 8 3" "1 8 4"; do
  set -- $cfg
  python -m paper_2407_14783_b200.build -D QB_DYN_PAIRS=$1 -D QB_DYN_MINB=$2 -D QB_DYN2_MINB=$3 > /dev/null 2>&1
  timeout 600 python bench.py --workload c1 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/k1_$1_$2_$3.log 2>&1; echo k1_$1_$2_$3=$?
done
python -m paper_2407_14783_b200.build --force > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_gradients.py -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
