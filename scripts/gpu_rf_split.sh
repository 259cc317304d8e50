mkdir -p gpurun_out
for cfg in "48 2" "96 1" "192 1" "24 4"; do
set -- $cfg
python -m paper_2407_14783_b200.build -D QB_RF_WANT=$1 -D QB_RF_TPW=$2 > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python bench.py --workload c2 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/c2.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/c2.log') if x.startswith('{')]
d=json.loads(l[-1]); print('want $1 tpw $2: c2', '%.4g'%d['value'], d['ms_per_step'])"
done
