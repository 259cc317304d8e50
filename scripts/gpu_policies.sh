# new policy tests on the GPU + the C3 bench line
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_policies.py tests/test_policies.py tests/test_quatmath.py -q -rf --tb=short -p no:cacheprovider > gpurun_out/pytest_pol.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_pol.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('roofline_render_issue'))"
