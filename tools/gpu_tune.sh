cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fill_kernel|brownian_steps|staged_prefix" -c 3 -o gpurun_out/prof_bm2 python tools/prof_kernels.py normal brownian prefix > gpurun_out/ncu_full.log 2>&1
