#!/bin/bash
# A/B of library variants (scripts/_dbg/<name>.so) on one workload (WL, default c5):
# prints value, per-kernel ms and the SM clock per variant
for v in "" "$@"; do
  if [ -z "$v" ]; then lib=""; name=default; else lib="scripts/_dbg/$v.so"; name=$v; fi
  QB_LIB_PATH=$lib python bench.py --workload ${WL:-c5} --steps ${STEPS:-10} --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value']), d.get('kernel_ms'), d.get('clocks',{}).get('sm_mhz'))"
done
