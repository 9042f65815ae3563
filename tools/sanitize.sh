#!/usr/bin/env bash
# compute-sanitizer over the C++ API tests, the device-lambda test and the
# kernel parity tests (minus the full-size cases); racecheck/synccheck on the
# TMA bulk kernel, whose shared-memory ring is the only smem producer/consumer.
# API errors are not reported: the error-mapping tests fail cudaMalloc and
# cudaSetDevice on purpose.
out=${1:-gpurun_out/sanitize}
mkdir -p "$out"
CS=/usr/local/cuda/bin/compute-sanitizer
L=paper_2206_06302_b200/lib
timeout 900 $CS --tool memcheck --report-api-errors no --leak-check full --error-exitcode 9 $L/test_api --gpu > "$out/memcheck_test_api.txt" 2>&1; echo "memcheck test_api rc=$?" >> "$out/rc.txt"
timeout 900 $CS --tool memcheck --error-exitcode 9 $L/test_lambda > "$out/memcheck_test_lambda.txt" 2>&1; echo "memcheck test_lambda rc=$?" >> "$out/rc.txt"
timeout 1500 $CS --tool memcheck --report-api-errors no --error-exitcode 9 python -m pytest tests/test_kernels_gpu.py -q -m gpu \
  -k "not full_size and not tuning_shapes" > "$out/memcheck_kernels.txt" 2>&1; echo "memcheck kernels rc=$?" >> "$out/rc.txt"
timeout 900 $CS --tool racecheck --error-exitcode 9 python -m pytest tests/test_kernels_gpu.py -q -m gpu \
  -k "tma_bulk and float64" > "$out/racecheck_tma.txt" 2>&1; echo "racecheck tma rc=$?" >> "$out/rc.txt"
timeout 900 $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_kernels_gpu.py -q -m gpu \
  -k "tma_bulk and float64" > "$out/synccheck_tma.txt" 2>&1; echo "synccheck tma rc=$?" >> "$out/rc.txt"
timeout 900 $CS --tool racecheck --error-exitcode 9 python -m pytest tests/test_kernels_gpu.py -q -m gpu \
  -k "experimental and float64" > "$out/racecheck_hybrid.txt" 2>&1; echo "racecheck hybrid rc=$?" >> "$out/rc.txt"
timeout 900 $CS --tool memcheck --report-api-errors no --error-exitcode 9 python -m pytest tests/test_kernels_gpu.py -q -m gpu \
  -k "pinned or probe or pageable" > "$out/memcheck_pinned_probes.txt" 2>&1; echo "memcheck pinned/probes rc=$?" >> "$out/rc.txt"
# round 2: tile chains (global flags, barriers around the flag waits),
# stream-ordered staging workers, per-target graphs, the NCCL rank path
timeout 1500 $CS --tool memcheck --report-api-errors no --error-exitcode 9 python -m pytest tests/test_stream_gpu.py -q -m gpu \
  -k "chain or pdl or pageable or stream_ordered or spans or stamps" > "$out/memcheck_chain_staging.txt" 2>&1; echo "memcheck chain/staging rc=$?" >> "$out/rc.txt"
timeout 1500 $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_stream_gpu.py -q -m gpu \
  -k "tile_chain" > "$out/synccheck_chain.txt" 2>&1; echo "synccheck chain rc=$?" >> "$out/rc.txt"
timeout 1500 $CS --tool memcheck --report-api-errors no --error-exitcode 9 python -m pytest tests/test_multigpu_gpu.py -q -m gpu \
  > "$out/memcheck_multigpu.txt" 2>&1; echo "memcheck multigpu rc=$?" >> "$out/rc.txt"
