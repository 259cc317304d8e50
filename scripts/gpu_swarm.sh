mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_swarm.py -q -rA --tb=short -p no:cacheprovider > gpurun_out/pytest_swarm.log 2>&1; echo swarm=$?
grep -E "^E  |Error|FAILED|passed|failed" gpurun_out/pytest_swarm.log | head -30
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
