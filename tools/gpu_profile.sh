# Profile session: launch list of the bench command + one full ncu capture per hot kernel,
# summarised on the box (the .ncu-rep is too large to bring back whole).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TAG=${PROFILE_TAG:-rX}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --quick --steps 2 --warmup 1 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"fill_kernel|normal_fill|staged_prefix|rowsplit|brownian_fused|brownian_steps" -c ${NCU_COUNT:-8} \
    -o /tmp/prof_full python tools/prof_kernels.py ${NCU_WHICH:-fill tyche prefix normal brownian} > gpurun_out/ncu_full.log 2>&1
python tools/summarize_profiles.py "$TAG" gpurun_out/launches.csv /tmp/prof_full.ncu-rep > gpurun_out/summarize.log 2>&1
mkdir -p gpurun_out/profiles
cp profiles/${TAG}_launches.md profiles/${TAG}_ncu.md profiles/ncu_summary.json gpurun_out/profiles/ 2>/dev/null
for k in "fill_kernel<(int)1, (int)1" "fill_kernel<(int)2, (int)1" "staged_prefix_kernel<(int)3" "normal_fill_kernel<(int)0"; do
    timeout 300 python tools/ncu_source.py /tmp/prof_full.ncu-rep "$k" 25 >> gpurun_out/profiles/${TAG}_stalls.txt 2>&1
done
rm -f gpurun_out/launches.csv
ls -la gpurun_out gpurun_out/profiles
