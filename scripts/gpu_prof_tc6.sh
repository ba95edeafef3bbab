#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
O=gpurun_out/proftc6; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_stage_kernel -s 6 -c 1 -o $O/prof_tc6 \
  python bench.py --order 6 --cells 40 40 40 --steps 1 --warmup 3 --extras none --no-cpu-baseline --e2e-steps 1 --dropin-steps 0 > $O/ncu.log 2>&1
tail -1 $O/ncu.log
