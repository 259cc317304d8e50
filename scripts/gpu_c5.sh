# C5 BVH renderer with camera frontier: parity + stats + register-cap variants
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_env.py -q -x -p no:cacheprovider > gpurun_out/pytest_render.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_render.log
python -m paper_2407_14783_b200.build -D QB_RF_STATS > gpurun_out/stats_build.log 2>&1; echo build=$?
timeout 300 python scripts/render_stats.py 8192 > gpurun_out/stats.log 2>&1; echo stats=$?
tail -2 gpurun_out/stats.log
for m in 24 20 18; do
  python -m paper_2407_14783_b200.build -D QB_RF_MINB=$m > /dev/null 2>&1
  timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/c5_$m.log 2>&1; echo c5_$m=$?
done
