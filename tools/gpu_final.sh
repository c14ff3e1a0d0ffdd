#!/bin/bash
# End-of-round evidence session (TAG): tests, smoke, bench (+2-rank gloo, reference arm), launch
# list + full ncu + stall dump, sanitizers, bench matrix, scalar latency. Everything to keep is
# copied to gpurun_out/profiles/ as ${TAG}_*.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out/profiles
TAG=${TAG:-r2z}
DO_MULTI=1 bash tools/gpu_round.sh
PROFILE_TAG=$TAG bash tools/gpu_profile.sh
bash tools/sanitize.sh
timeout 900 python tools/bench_matrix.py > gpurun_out/bench_matrix.json 2> gpurun_out/bench_matrix.err
timeout 900 python tools/bench_scalar.py > gpurun_out/scalar.json 2> gpurun_out/scalar.err
P=gpurun_out/profiles
cp gpurun_out/bench.json $P/${TAG}_bench.json
cp gpurun_out/bench_2rank.json $P/${TAG}_bench_2rank_gloo_1gpu.json
cp gpurun_out/bench_ref.json $P/${TAG}_bench_reference.json
cp gpurun_out/bench_matrix.json $P/${TAG}_bench_matrix.json
cp gpurun_out/scalar.json $P/${TAG}_scalar.json
cp gpurun_out/sanitize_memcheck.log $P/${TAG}_sanitize_memcheck.log
cp gpurun_out/sanitize_racecheck.log $P/${TAG}_sanitize_racecheck.log
tail -5 gpurun_out/pytest_gpu.log > $P/${TAG}_pytest_gpu_tail.txt
cat gpurun_out/smoke.log >> $P/${TAG}_pytest_gpu_tail.txt
ls -la $P
