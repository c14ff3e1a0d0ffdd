#!/bin/bash
# r2g session: split-mulhilo Philox in the Box-Muller fill: parity, timings, ncu.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "normal2 or box or cfg3" > gpurun_out/t_r2g.log 2>&1; echo rc=$? >> gpurun_out/t_r2g.log
timeout 1200 python -m pytest tests/test_gpu_variants.py -q -p no:cacheprovider -k "LAYOUT or SPLIT" >> gpurun_out/t_r2g.log 2>&1; echo rc=$? >> gpurun_out/t_r2g.log
TUNE_SETS="CBRNG_BM_SPLIT=0;CBRNG_BM_LAYOUT=5;CBRNG_BM_LAYOUT=12;CBRNG_BM_LAYOUT=9;CBRNG_BM_LAYOUT=4;CBRNG_BM_LAYOUT=0;CBRNG_BM_LAYOUT=2;CBRNG_BM_LAYOUT=8" timeout 900 python tools/tune_bm.py > gpurun_out/tune_bm.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"normal_fill" -c 1 -o gpurun_out/prof_r2g python tools/prof_kernels.py normal > gpurun_out/ncu_r2g.log 2>&1
