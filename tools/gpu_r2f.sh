#!/bin/bash
# r2f session: software-pipelined Box-Muller layouts: variant parity, timings, ncu.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_variants.py -q -p no:cacheprovider -k "LAYOUT" > gpurun_out/t_r2f.log 2>&1; echo rc=$? >> gpurun_out/t_r2f.log
TUNE_SETS="CBRNG_BM_LAYOUT=5;CBRNG_BM_LAYOUT=8;CBRNG_BM_LAYOUT=9;CBRNG_BM_LAYOUT=10;CBRNG_BM_LAYOUT=11;CBRNG_BM_LAYOUT=12;CBRNG_BM_LAYOUT=9,CBRNG_BM_GRID=2" timeout 900 python tools/tune_bm.py > gpurun_out/tune_bm.jsonl 2>&1
CBRNG_BM_LAYOUT=9 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"normal_fill" -c 1 -o gpurun_out/prof_r2f python tools/prof_kernels.py normal --tuning > gpurun_out/ncu_r2f.log 2>&1
