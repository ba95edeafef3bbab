#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out/tune2
for v in base g4e1; do
  lib=$PWD/paper_0901_1024_b200/libdgm_$v.so; [ "$v" = base ] && lib=$PWD/paper_0901_1024_b200/libdgm.so
  for n in 1 2 3 5 7 8 9; do
    DGM_LIB=$lib timeout 300 python bench.py --order $n --cells 20 20 20 --dtype f64 --steps 6 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/tune2/${v}_n$n.json 2> gpurun_out/tune2/${v}_n$n.err
  done
done
echo done
