cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
TUNE_GRID=8 TUNE_ILP=4,2 TUNE_TF=2 timeout 900 python tools/tune_fills.py > gpurun_out/tune.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fill_kernel<2|tyche_prefix" -c 2 -o gpurun_out/prof_sq python tools/prof_kernels.py fill tyche > gpurun_out/ncu_full.log 2>&1
