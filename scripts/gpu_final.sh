# end-of-session check: smoke + GPU suite + default bench + reference arm
mkdir -p gpurun_out
bash scripts/gpu_tests.sh
timeout 600 python bench.py > gpurun_out/bench_final.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_final.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d.get('roofline_render_issue',{}).get('frac'), d['cpu_baseline']['value'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
tail -1 gpurun_out/bench_ref.log | cut -c1-400
