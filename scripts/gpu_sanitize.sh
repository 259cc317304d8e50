mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_kernels.py tests/test_gpu_noise.py tests/test_gpu_swarm.py tests/test_gpu_dropin.py \
  -q -x -p no:cacheprovider -k "not fp32_close and not episode" > gpurun_out/memcheck.log 2>&1; echo memcheck=$?
tail -15 gpurun_out/memcheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/racecheck.log 2>&1; echo racecheck=$?
tail -6 gpurun_out/racecheck.log
