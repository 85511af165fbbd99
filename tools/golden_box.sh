#!/bin/bash
# Generate the 8000² golden on the GPU box's host (196 GB RAM; this container
# has 62 GB, too little for the reference's 31 GB basis + two CSR copies).
# Runs the prebuilt reference (oracle/_ref) in both builds side by side;
# the outputs are merged into tests/golden/solver_golden.json by
# tools/golden_merge.py in the container.
set -u
mkdir -p gpurun_out
KRY_REF_VARIANT=ref timeout 3600 python tests/golden/make_golden.py --solve-json two_2d8000_s60_c1 > gpurun_out/golden8000_ref.json 2> gpurun_out/golden8000_ref.err &
KRY_REF_VARIANT=fma timeout 3600 python tests/golden/make_golden.py --solve-json two_2d8000_s60_c1 > gpurun_out/golden8000_fma.json 2> gpurun_out/golden8000_fma.err &
wait
ls -la gpurun_out/golden8000_*
