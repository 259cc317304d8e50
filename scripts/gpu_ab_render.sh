# A/B of a workload (WL=c3 default) between library builds in scripts/_dbg (VARIANTS, default "base new"), alternating
WL=${WL:-c3}
STEPS=${STEPS:-30}
for r in 1 2 3; do
  for v in ${VARIANTS:-base new}; do
    QB_LIB_PATH=$PWD/scripts/_dbg/$v.so timeout 300 python bench.py --workload $WL --steps $STEPS --warmup 3 --no-e2e --no-cpu --no-sub > gpurun_out/ab_$v.log 2>&1
    python -c "
import json
l=[x for x in open('gpurun_out/ab_$v.log') if x.startswith('{')]
d=json.loads(l[-1]); km=d.get('kernel_ms', {}); print('$v', 'value %.4g'%d['value'], 'render %.4f ms'%km.get('render_k2', -1), 'step %.4f'%d['ms_per_step'], ' '.join('%s %.4f'%(k, x) for k, x in km.items() if k != 'render_k2'))"
  done
done
