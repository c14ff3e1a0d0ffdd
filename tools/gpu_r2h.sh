#!/bin/bash
# r2h session: HBM-free ceilings (CBRNG_NOSTORE: stores into an L2-resident ring) of the fills and Box-Muller.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TUNE_SETS="CBRNG_NOSTORE=0;CBRNG_NOSTORE=1" timeout 900 python tools/tune_fills.py > gpurun_out/tune_fills.log 2>&1
TUNE_SETS="CBRNG_NOSTORE=0;CBRNG_NOSTORE=1" timeout 900 python tools/tune_bm.py > gpurun_out/tune_bm.jsonl 2>&1
