mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --tb=short -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "^E  |FAILED|passed|failed" gpurun_out/pytest_gpu.log | head -5
for pf in 1 0; do
python -m paper_2407_14783_b200.build -D QB_ENV_PF=$pf > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
echo "pf $pf: $(PYTHONPATH=. timeout 300 python scripts/envstep_time.py 2>&1 | tail -1)"
done
