mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_noise.py -q -rA --tb=short -p no:cacheprovider > gpurun_out/pytest_noise.log 2>&1; echo noise=$?
tail -30 gpurun_out/pytest_noise.log
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
