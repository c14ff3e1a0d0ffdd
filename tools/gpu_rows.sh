cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_variants.py -q -p no:cacheprovider -k "rows256" > gpurun_out/t.log 2>&1; echo rc=$? >> gpurun_out/t.log
for r in 1 2; do for l in 0 4 8 16; do for a in philox threefry; do echo "split=$l $(CBRNG_MS_SPLIT=$l python tools/probes/probe_rows.py $a --tuning)" >> gpurun_out/rows.txt; done; done; done
