#!/bin/bash
# r2c session: BM front-end parity, Brownian per-warp step table (parity + timing).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "normal2 or Brownian" -p no:cacheprovider > gpurun_out/t_r2c.log 2>&1; echo rc=$? >> gpurun_out/t_r2c.log
timeout 900 python -m pytest tests/test_gpu_variants.py -q -k "misc" -p no:cacheprovider >> gpurun_out/t_r2c.log 2>&1; echo rc=$? >> gpurun_out/t_r2c.log
TUNE_SETS="CBRNG_BM_MINB=8;CBRNG_BM_MINB=0" timeout 600 python tools/tune_bm.py > gpurun_out/tune_bm.jsonl 2>&1
for t in 1 2 1 2; do CBRNG_BROWNIAN_TAB=$t timeout 300 python tools/tune_brownian.py >> gpurun_out/tune_br.jsonl 2>&1; echo "tab=$t" >> gpurun_out/tune_br.jsonl; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"brownian_fused" -c 1 -o gpurun_out/prof_br python tools/prof_kernels.py brownian > gpurun_out/ncu_br.log 2>&1
