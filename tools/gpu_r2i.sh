#!/bin/bash
# r2i session: Squares round forms (CBRNG_SQ_INC=1..4): variant parity, timings.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -q -p no:cacheprovider -k "squares_round1" > gpurun_out/t_r2i.log 2>&1; echo rc=$? >> gpurun_out/t_r2i.log
TUNE_SETS="CBRNG_SQ_INC=1;CBRNG_SQ_INC=2;CBRNG_SQ_INC=3;CBRNG_SQ_INC=4;CBRNG_SQ_INC=2,CBRNG_FILL_ILP=12;CBRNG_SQ_INC=4,CBRNG_FILL_ILP=12" timeout 900 python tools/tune_fills.py > gpurun_out/tune_fills.log 2>&1
