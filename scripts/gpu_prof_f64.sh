#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
O=gpurun_out/proff64; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 6 -c 1 -o $O/prof_f64_c3 \
  python bench.py --dtype f64 --steps 1 --warmup 3 --extras none --no-cpu-baseline --e2e-steps 1 --dropin-steps 0 > $O/ncu.log 2>&1
tail -2 $O/ncu.log
