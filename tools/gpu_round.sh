#!/bin/bash
# One GPU session: tests, smoke, bench (+ multi-rank logic check, reference arm), optional ncu.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/nproc.txt
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 ${PYTEST_ARGS:-} -s --durations=25 -p no:cacheprovider -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
if [ -n "$DO_MULTI" ]; then
  timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --no-cpu \
      > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
  echo "2rank rc=$?" >> gpurun_out/bench_2rank.err
  timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
fi
if [ -n "$DO_NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --quick --steps 2 --warmup 1 > gpurun_out/ncu_launch_bench.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_KERNELS:-fill_kernel|tyche_prefix|prefix_kernel|brownian_steps}" -c ${NCU_COUNT:-8} -o gpurun_out/prof_full python tools/prof_kernels.py ${NCU_WHICH:-fill tyche prefix normal brownian} > gpurun_out/ncu_full.log 2>&1
fi
ls -la gpurun_out
