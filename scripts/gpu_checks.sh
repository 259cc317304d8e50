# Memory / race checks without compute-sanitizer (closed on this pool): the checked build
# (-DQB_CHECKS: kernels assert their own index arithmetic, csrc/qb_checks.cuh), built locally by
#   bash scripts/build_variant.sh checks -DQB_CHECKS
# and shipped in scripts/_dbg/checks.so; runs scripts/checks.py (output coverage, determinism,
# split-vs-batch renders, adjoint reproducibility), the kernel-family cases and the GPU suite with it.
mkdir -p gpurun_out
export QB_LIB_PATH=$PWD/scripts/_dbg/checks.so
python scripts/checks.py > gpurun_out/checks.log 2>&1; echo checks=$?
python scripts/sanitize_cases.py env grad query bindings > gpurun_out/checks_cases.log 2>&1; echo cases=$?
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/checks_pytest.log 2>&1; echo pytest=$?
tail -1 gpurun_out/checks_pytest.log
echo "QB_CHECK failures: $(cat gpurun_out/checks.log gpurun_out/checks_cases.log gpurun_out/checks_pytest.log | grep -c 'QB_CHECK FAILED')"
grep -E "^(ok|FAIL)|checks:" gpurun_out/checks.log
