#!/bin/bash
# A/B of a bench.py flag: default vs "$FLAG" on the workload in $BENCH_ARGS, interleaved twice.
# Usage: FLAG="--face-slots natural" BENCH_ARGS="--order 6 --cells 20 20 20" bash scripts/gpu_flag_ab.sh tag
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
O=gpurun_out/flag_$1; mkdir -p $O
for rep in 1 2; do
  timeout 300 python bench.py $BENCH_ARGS --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 > $O/default_$rep.json 2> $O/default_$rep.err
  timeout 300 python bench.py $BENCH_ARGS $FLAG --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 > $O/flag_$rep.json 2> $O/flag_$rep.err
done
