# full GPU parity suite + the env-step and sensor-pass timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --tb=short -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "^E  |FAILED|passed|failed" gpurun_out/pytest_gpu.log | head -10
PYTHONPATH=. timeout 300 python scripts/envstep_time.py 2>&1 | tail -1
timeout 600 python bench.py --workload c3n --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/c3n.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/c3n.log') if x.startswith('{')]
d=json.loads(l[-1]); print('c3n', '%.4g'%d['value'], d.get('kernel_ms'))"
