cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TUNE_GRID=8 TUNE_ILP=8,4 TUNE_TF=2 timeout 900 python tools/tune_fills.py > gpurun_out/tune.log 2>&1
bash tools/sanitize.sh
