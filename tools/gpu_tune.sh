cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
TUNE_GRID=8,16 TUNE_ILP=16,8 TUNE_TF=2 timeout 900 python tools/tune_fills.py > gpurun_out/tune.log 2>&1
