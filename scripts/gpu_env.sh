# env kernels (warp-per-env small batches): parity + c1/c2/c3
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for w in c1 c2 c3 c1 c2; do
timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/$w.log 2>&1; echo $w=$?
python -c "
import json
l=[x for x in open('gpurun_out/$w.log') if x.startswith('{')]
d=json.loads(l[-1]); print('$w', '%.4g'%d['value'], d.get('kernel_ms'), d['ms_per_step'])"
done
