#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out/oab
for o in natural columns; do
  timeout 600 python bench.py --dtype f64 --steps 6 --warmup 3 --e2e-steps 1 --no-cpu-baseline --element-order $o > gpurun_out/oab/f64_$o.json 2>/dev/null
  for n in 7 8 9; do
    timeout 300 python bench.py --order $n --cells 20 20 20 --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline --element-order $o > gpurun_out/oab/n${n}_$o.json 2>/dev/null
  done
done
echo done
