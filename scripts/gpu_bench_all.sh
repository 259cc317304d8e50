mkdir -p gpurun_out
for w in c3 c1 c2 c2a c4 c5 c3n swarm; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.log 2>&1; echo bench_$w=$?
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
tail -1 gpurun_out/bench_ref.log
PYTHONPATH=. timeout 300 python scripts/scene_build_bench.py > gpurun_out/scene_build.log 2>&1; echo scene_build=$?
PYTHONPATH=. timeout 300 python scripts/envstep_time.py > gpurun_out/envstep.log 2>&1; echo envstep=$?
