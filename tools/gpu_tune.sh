cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TUNE_GRID=2,4,8,16 TUNE_ILP=4 timeout 900 python tools/tune_fills.py > gpurun_out/tune.log 2>&1
TUNE_GRID=4,8 TUNE_ILP=2 timeout 900 python tools/tune_fills.py >> gpurun_out/tune.log 2>&1
