mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -k "rollout or bptt or grad or adjoint or vjp or autograd" -q -rf --tb=short -p no:cacheprovider > gpurun_out/pytest_c4.log 2>&1; echo pytest=$?
grep -E "^E  |FAILED|passed|failed" gpurun_out/pytest_c4.log | head -10
for r in 1 2; do
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/c4.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/c4.log') if x.startswith('{')]
d=json.loads(l[-1]); print('c4', '%.4g'%d['value'], d.get('kernel_ms'))"
done
