# GPU parity suite + smoke (used from gpurun)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q -rA --tb=short -p no:cacheprovider -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
python scripts/debug_landing.py > gpurun_out/debug_landing.log 2>&1
