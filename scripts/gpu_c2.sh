mkdir -p gpurun_out
bash scripts/gpu_one.sh tests/test_gpu_edges.py
for w in c2 c2a; do
timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e > gpurun_out/$w.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/$w.log') if x.startswith('{')]
d=json.loads(l[-1]); print('$w', '%.4g'%d['value'], d['ms_per_step'], 'cpu', (d.get('cpu_baseline') or {}).get('value'))"
done
