mkdir -p gpurun_out
python -m paper_2407_14783_b200.build -D QB_RF_STATS -D QB_RF_WIDE=0 > gpurun_out/stats_build.log 2>&1; echo build=$?
timeout 300 python scripts/render_stats.py 8192 > gpurun_out/stats.log 2>&1; echo stats=$?
cat gpurun_out/stats.log | tail -5
