#!/bin/bash
# Final round-1 numbers: C3 fp64, C4 (8M tets, N=4), C5 (N=6, 2.06M tets) on one B200.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out/final
timeout 600 python bench.py --dtype f64 --steps 10 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/final/c3_f64.json 2> gpurun_out/final/c3_f64.err
timeout 1200 python bench.py --cells 110 110 110 --steps 10 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/final/c4.json 2> gpurun_out/final/c4.err
timeout 900 python bench.py --order 6 --cells 70 70 70 --steps 10 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/final/c5.json 2> gpurun_out/final/c5.err
echo done
