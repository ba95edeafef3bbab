#!/bin/bash
# C4 (8M tets, N=4) and C5 (N=6, 2.06M tets) on one B200.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out/big
free -g > gpurun_out/big/host_mem.txt; nproc >> gpurun_out/big/host_mem.txt
timeout 1200 python bench.py --cells 110 110 110 --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/big/c4.json 2> gpurun_out/big/c4.err
timeout 900 python bench.py --order 6 --cells 70 70 70 --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/big/c5.json 2> gpurun_out/big/c5.err
echo done
