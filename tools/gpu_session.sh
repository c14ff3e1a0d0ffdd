# One GPU session: full GPU tests, a tune pass (TUNE_SETS), the bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x -rA --junitxml=gpurun_out/pytest_gpu.xml > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
if [ -n "$TUNE_SETS" ]; then timeout 900 python tools/tune_fills.py > gpurun_out/tune.log 2>&1; fi
timeout 900 python bench.py ${BENCH_ARGS:---steps 50 --warmup 3} > gpurun_out/bench.json 2> gpurun_out/bench.err
