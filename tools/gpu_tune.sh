# Variant sweep session: parity of every variant, then timings (tools/tune_fills.py).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_variants.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_variants.log
TUNE_SETS="${TUNE_SETS:-}" timeout 1500 python tools/tune_fills.py > gpurun_out/tune.log 2>&1
