mkdir -p gpurun_out
timeout 600 python -m pytest $@ -q -rf --tb=short -p no:cacheprovider > gpurun_out/pytest_one.log 2>&1; echo pytest=$?
grep -E "^E  |FAILED|passed|failed" gpurun_out/pytest_one.log | head -20
