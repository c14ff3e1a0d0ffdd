cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
TUNE_SETS="CBRNG_BM_MINB=0;CBRNG_BM_MINB=5;CBRNG_BM_MINB=6;CBRNG_BM_MINB=8" timeout 900 python tools/tune_fills.py > gpurun_out/tune.log 2>&1
timeout 900 python bench.py --steps 50 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
