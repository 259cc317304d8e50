# GPU parity suite + smoke (used from gpurun)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q -rf --tb=short -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "^E  |FAILED|passed|failed" gpurun_out/pytest_gpu.log | head -20
