mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --tb=short -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "^E  |FAILED|passed|failed" gpurun_out/pytest_gpu.log | head -5
for w in c1 c2a c2; do
for r in 1 2; do
timeout 600 python bench.py --workload $w --steps 100 --warmup 3 --no-e2e --no-cpu > gpurun_out/$w.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/$w.log') if x.startswith('{')]
d=json.loads(l[-1]); print('$w', '%.4g'%d['value'], '%.4g ms'%d['ms_per_step'])"
done
done
