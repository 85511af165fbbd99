#!/bin/bash
# compute-sanitizer over a small-size slice of the GPU suite (run on the GPU
# box: bash tools/sanitize.sh; logs in gpurun_out/sanitize_*.log).
# memcheck: out-of-bounds / misaligned device accesses and leaks;
# racecheck: shared-memory hazards; synccheck: illegal barrier use.
set -u
SEL='test_laplace2d_stencil_bitwise or test_laplace3d_stencil_bitwise or test_csr_spmv_bitwise or test_mpk_fused_bitwise or test_mpk3d_fused_bitwise or test_gram_matches_reference or test_bcgs_pip_matches_reference or test_jacobi'
SOLVE='pip2_2d16 or two_2d64_s60 or two_3d16_s60 or two_2d48_csr or standard_2d32'
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  timeout 2400 compute-sanitizer --tool $tool $extra --target-processes all --error-exitcode 99 \
    python -m pytest -q -x -p no:cacheprovider tests/test_gpu_kernels.py -k "$SEL and not 100003 and not 512 and not 256" \
    > gpurun_out/sanitize_${tool}_kernels.log 2>&1
  echo "EXIT=$?" >> gpurun_out/sanitize_${tool}_kernels.log
  timeout 2400 compute-sanitizer --tool $tool $extra --target-processes all --error-exitcode 99 \
    python -m pytest -q -x -p no:cacheprovider tests/test_gpu_solver.py -k "test_solver_matches_reference and ($SOLVE) and not fused" \
    > gpurun_out/sanitize_${tool}_solver.log 2>&1
  echo "EXIT=$?" >> gpurun_out/sanitize_${tool}_solver.log
done
