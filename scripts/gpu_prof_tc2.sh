#!/bin/bash
# ncu --set full (with source) of the v2 stage kernel at C3, an LSRK stage with a != 0.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
O=gpurun_out/proftc2; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc2_stage_kernel -s 6 -c 1 -o $O/prof_tc2_c3 \
  python bench.py --steps 1 --warmup 3 --extras none --no-cpu-baseline --e2e-steps 1 --dropin-steps 0 --path tensor2 > $O/ncu.log 2>&1
tail -3 $O/ncu.log
