mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --tb=short -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "^E  |FAILED|passed|failed" gpurun_out/pytest_gpu.log | head -10
for r in 1 2 3; do
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/c3.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/c3.log') if x.startswith('{')]
d=json.loads(l[-1]); print('c3', '%.4g'%d['value'], d.get('kernel_ms'))"
done
