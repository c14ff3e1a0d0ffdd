#!/bin/bash
# r2d session: Squares ALU-forced carries + Box-Muller 6-op sqrt / pi/512 sincos table:
# parity, variant parity, timings.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "squares or Squares or normal2 or box or cfg3 or cfg1" > gpurun_out/t_r2d.log 2>&1; echo rc=$? >> gpurun_out/t_r2d.log
timeout 1200 python -m pytest tests/test_gpu_variants.py -q -p no:cacheprovider -k "squares or misc or ilp" >> gpurun_out/t_r2d.log 2>&1; echo rc=$? >> gpurun_out/t_r2d.log
TUNE_SETS="CBRNG_FILL_ILP=16;CBRNG_FILL_ILP=12;CBRNG_SQ_MINB=6,CBRNG_FILL_ILP=16;CBRNG_SQ_MINB=6,CBRNG_FILL_ILP=12" timeout 900 python tools/tune_fills.py > gpurun_out/tune_fills.log 2>&1
TUNE_SETS="CBRNG_BM_MINB=8;CBRNG_BM_MINB=0;CBRNG_BM_ILP=6;CBRNG_BM_ILP=6,CBRNG_BM_MINB=0;CBRNG_BM_ILP=4;CBRNG_BM_ILP=4,CBRNG_BM_MINB=0" timeout 900 python tools/tune_bm.py > gpurun_out/tune_bm.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fill_kernel" -c 2 -o gpurun_out/prof_r2d python tools/prof_kernels.py normal squares > gpurun_out/ncu_r2d.log 2>&1
