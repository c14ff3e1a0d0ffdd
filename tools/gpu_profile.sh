# Profile session: launch list of the bench command + one full ncu capture per hot kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --quick --steps 2 --warmup 1 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"fill_kernel|staged_prefix|brownian_fused|brownian_steps" -c ${NCU_COUNT:-8} \
    -o gpurun_out/prof_full python tools/prof_kernels.py ${NCU_WHICH:-fill tyche prefix normal brownian} > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
