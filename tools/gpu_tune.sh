cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "Brownian" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for m in 5 6; do echo "MINB=$m $(CBRNG_BROWNIAN_MINB=$m timeout 600 python tools/tune_brownian.py 2>&1 | tail -1)" >> gpurun_out/tune.log; done
