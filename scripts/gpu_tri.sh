mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --tb=short -p no:cacheprovider -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "^E  |FAILED|passed|failed|mesh config 2" gpurun_out/pytest_gpu.log | head -10
for w in c5 c2; do
timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/$w.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/$w.log') if x.startswith('{')]
d=json.loads(l[-1]); print('$w', '%.4g'%d['value'], d['ms_per_step'], d.get('kernel_ms'))"
done
