mkdir -p gpurun_out
for cfg in "8 4" "8 6" "8 8" "4 6" "16 6"; do
set -- $cfg
python -m paper_2407_14783_b200.build -D QB_OBS_UNROLL=$1 -D QB_OBS_MINB=$2 > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -5 gpurun_out/build.log; exit 1; }
timeout 600 python bench.py --workload c3n --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/c3n.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/c3n.log') if x.startswith('{')]
d=json.loads(l[-1]); print('c3n $1 $2', '%.4g'%d['value'], d.get('kernel_ms'))"
done
python -m paper_2407_14783_b200.build --force > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_noise.py -q -p no:cacheprovider > gpurun_out/pytest_noise.log 2>&1; echo noise=$?; tail -1 gpurun_out/pytest_noise.log
