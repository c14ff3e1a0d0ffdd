#!/bin/bash
# compute-sanitizer memcheck + racecheck over the small-size parity tests (GPU box).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
SEL='edge_sizes or row_shapes or resume_mid_block or random_streams or prefix_uniform or vector_ciphers or checksum_1000 or cases_bit_exact or histograms_exact or avalanche_exact or tyche_fill or normal2_within or normal2_words_edges or mixed_scalar or chunked_steps or restart or packed_records'
timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_battery.py tests/test_gpu_scalar.py -m gpu -q -p no:cacheprovider \
    -k "$SEL or philox_block or tyche_words or generator_windows" \
    > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/sanitize_memcheck.log
timeout 1800 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_battery.py -m gpu -q -p no:cacheprovider \
    -k "row_shapes or random_streams or prefix_uniform or histograms_exact or interleave or normal2_within or normal2_words_edges or chunked_steps" \
    > gpurun_out/sanitize_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/sanitize_racecheck.log
