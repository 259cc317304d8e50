for r in 1 2 3; do
timeout 600 python bench.py --workload c3 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/c3.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/c3.log') if x.startswith('{')]
d=json.loads(l[-1]); print('c3', '%.4g'%d['value'], d.get('kernel_ms'))"
done
