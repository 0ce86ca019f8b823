#!/bin/bash
# Final-code evidence run on the GPU box: compute-sanitizer memcheck over the parity / streaming /
# warp-kernel tests (everything but the full-size and sub-process tests), racecheck over the
# shared-memory kernels, then the randomized differential runs (C ABI and C++ adapter).
# usage: bash tools/run_final_checks.sh [fuzz seconds] [adapter fuzz seconds]
FUZZ=${1:-600}
AFUZZ=${2:-120}
mkdir -p gpurun_out
SKIP='not full_size and not 2pow and not large_batch and not huge and not reentrant and not pageable and not pipelined and not chunks_by_bytes and not in_pieces and not every_kernel_variant and not cuda_graph'
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -x -m gpu \
    tests/test_gpu_parity.py tests/test_gpu_streaming.py tests/test_gpu_warp_kernel.py -k "$SKIP" \
    > gpurun_out/final_memcheck.log 2>&1
echo "memcheck rc=$?"; tail -4 gpurun_out/final_memcheck.log
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -x -m gpu \
    tests/test_gpu_parity.py -k "pipelined or chunks_by_bytes or in_pieces or pageable or empty_messages" \
    > gpurun_out/final_memcheck_host.log 2>&1
echo "memcheck host rc=$?"; tail -4 gpurun_out/final_memcheck_host.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest -q -x -m gpu \
    tests/test_gpu_parity.py -k "bucket_order or all_short_ragged or variable_length_workload or lanesplit" \
    > gpurun_out/final_racecheck.log 2>&1
echo "racecheck rc=$?"; tail -4 gpurun_out/final_racecheck.log
python tests/fuzz_parity.py $FUZZ 29 > gpurun_out/final_fuzz.log 2>&1
echo "fuzz rc=$?"; tail -3 gpurun_out/final_fuzz.log; cp gpurun_out/fuzz_parity.json gpurun_out/final_fuzz_parity.json
tests/cpp/fuzz_batch_adapter $AFUZZ 31 20 > gpurun_out/final_adapter_fuzz.json 2> gpurun_out/final_adapter_fuzz.err
echo "adapter fuzz rc=$?"; tail -c 600 gpurun_out/final_adapter_fuzz.json
