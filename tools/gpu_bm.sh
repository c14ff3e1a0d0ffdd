#!/bin/bash
# Box-Muller session: parity + variant tests, variant timings, one full ncu capture.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "normal2" -p no:cacheprovider > gpurun_out/t_bm.log 2>&1; echo rc=$? >> gpurun_out/t_bm.log
timeout 900 python -m pytest tests/test_gpu_variants.py -q -k "misc" -p no:cacheprovider >> gpurun_out/t_bm.log 2>&1; echo rc=$? >> gpurun_out/t_bm.log
TUNE_SETS="CBRNG_BM_WS=0;CBRNG_BM_WS=1;CBRNG_BM_WS=2;CBRNG_BM_WS=3;CBRNG_BM_WS=4" timeout 900 python tools/tune_bm.py > gpurun_out/tune_bm.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bm_ws|fill_kernel" -c 1 -o gpurun_out/prof_bm python tools/prof_kernels.py normal > gpurun_out/ncu_bm.log 2>&1
