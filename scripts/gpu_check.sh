mkdir -p gpurun_out
bash scripts/gpu_tests.sh
for w in c2 c3; do
timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/$w.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/$w.log') if x.startswith('{')]
d=json.loads(l[-1]); print('$w', '%.4g'%d['value'], d.get('kernel_ms'))"
done
