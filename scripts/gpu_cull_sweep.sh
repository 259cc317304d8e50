mkdir -p gpurun_out
for cfg in "5 64 128" "6 56 64" "6 64 64" "6 48 64" "7 56 64"; do
set -- $cfg
python -m paper_2407_14783_b200.build -D QB_CULL_MINB=$1 -D QB_CREC=$2 -D QB_TPL_MAX=$3 > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -3 gpurun_out/build.log; exit 1; }
timeout 600 python bench.py --workload c3 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/c3.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/c3.log') if x.startswith('{')]
d=json.loads(l[-1]); print('c3 $1 $2 $3', '%.4g'%d['value'], d.get('kernel_ms'))"
done
