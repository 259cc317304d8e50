mkdir -p gpurun_out
for m in 4 5 1; do
python -m paper_2407_14783_b200.build -D QB_ENV_MINB=$m > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python bench.py --workload c1 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/c1.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/c1.log') if x.startswith('{')]
d=json.loads(l[-1]); print('env $m', '%.4g'%d['value'], d['roofline_env_step']['frac'], d['roofline_env_step']['ms'])"
done
python -m paper_2407_14783_b200.build --force > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_env.py tests/test_gpu_swarm.py tests/test_gpu_noise.py -q -p no:cacheprovider > gpurun_out/pytest_env.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_env.log
