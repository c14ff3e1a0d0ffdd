cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/probe_store.py > gpurun_out/probe_store.log 2>&1
timeout 900 python tools/tune_fills.py > gpurun_out/tune.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fill_kernel" -c 2 -o gpurun_out/prof_bm python tools/prof_kernels.py normal > gpurun_out/ncu_full.log 2>&1
