#!/bin/bash
# compute-sanitizer over the device kernels, ONE tool per invocation (per gpurun
# call; B200_PROFILING.md): scripts/sanitize.sh memcheck|racecheck|synccheck|initcheck
#
# Runs the small GPU parity tests that reach every kernel family: fused CG /
# FOM loops (entry, SpMV+dots, update with the ticket combine, finish, direction
# with the CGS sweeps), the fused F^{-1} tail (m <= 64) and the wide mu solve
# (m > 256), the stepped driver, SSOR's spin-wait sweeps, the 3x3-block and
# scalar SELL SpMV / SpMM, the DMMA Gram / GEMM and their split reductions, and
# the POD weighted Gram / coefficients. Output: gpurun_out/sanitize_<tool>.log
# plus a one-line summary in gpurun_out/sanitize_<tool>.summary.
set -u
tool=${1:?tool}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
log=gpurun_out/sanitize_${tool}.log
extra=""
[ "$tool" = "memcheck" ] && extra="--leak-check no"
sel='test_gpu_krylov.py tests/test_gpu_kernels.py tests/test_gpu_sequence.py tests/test_gpu_strategies.py'
kexpr='not c3_size and not fullsize and not concurrent and not c2_c3_like and not c1_poisson'
timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool "$tool" $extra --print-limit 50 --error-exitcode 99 \
  python -m pytest tests/$sel -m gpu -q -x -p no:cacheprovider -k "$kexpr" > "$log" 2>&1
rc=$?
errs=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" "$log" | tail -1)
passed=$(grep -E "passed|failed" "$log" | tail -1)
echo "{\"tool\": \"$tool\", \"rc\": $rc, \"summary\": \"$errs\", \"pytest\": \"$passed\"}" | tee gpurun_out/sanitize_${tool}.summary
