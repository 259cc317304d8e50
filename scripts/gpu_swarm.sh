mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_swarm.py tests/test_gpu_dropin.py tests/test_gpu_kernels.py -q -rf --tb=short -p no:cacheprovider > gpurun_out/pytest_swarm.log 2>&1; echo swarm=$?
grep -E "^E  |FAILED|passed|failed" gpurun_out/pytest_swarm.log | head -10
for w in swarm c3; do
timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/$w.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/$w.log') if x.startswith('{')]
d=json.loads(l[-1]); print('$w', '%.4g'%d['value'], d['ms_per_step'], d.get('kernel_ms'))"
done
