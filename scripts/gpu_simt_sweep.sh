#!/bin/bash
# SIMT stage kernel sweep: fp32 N=1..9 and fp64 N=4 at 48k tets, fp64 C3.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
out=gpurun_out/simt_${1:-x}; mkdir -p $out
for n in 1 2 3 4 5 6 7 8 9; do
  timeout 300 python bench.py --order $n --cells 20 20 20 --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline --path simt > $out/n$n.json 2> $out/n$n.err
done
for n in 4 6 9; do
  timeout 300 python bench.py --order $n --cells 20 20 20 --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline --dtype f64 > $out/d$n.json 2> $out/d$n.err
done
echo done
