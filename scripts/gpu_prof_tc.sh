#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_stage_kernel -s 5 -c 1 \
  -o gpurun_out/prof_tc python bench.py --steps 2 --warmup 3 --e2e-steps 1 --dropin-steps 0 --no-cpu-baseline --cells 30 30 30 > gpurun_out/ncu_tc.log 2>&1
echo done
