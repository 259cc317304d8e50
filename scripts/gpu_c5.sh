mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dropin.py -q -x -p no:cacheprovider > gpurun_out/pytest_render.log 2>&1; echo pytest=$?
tail -1 gpurun_out/pytest_render.log
for m in 24 20; do
python -m paper_2407_14783_b200.build -D QB_RF_MINB=$m > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/c5_$m.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/c5_$m.log') if x.startswith('{')]
d=json.loads(l[-1]); print('c5 $m', '%.4g'%d['value'], d.get('kernel_ms'))"
done
