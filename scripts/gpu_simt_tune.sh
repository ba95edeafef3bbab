#!/bin/bash
# fp64 SIMT kernel tuning: element groups G x elements per thread E (build overrides).
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out/tune
for v in base g8e1 g16e1 g4e2 g4e1; do
  lib=$PWD/paper_0901_1024_b200/libdgm_$v.so; [ "$v" = base ] && lib=$PWD/paper_0901_1024_b200/libdgm.so
  for n in 4 6; do
    DGM_LIB=$lib timeout 300 python bench.py --order $n --cells 20 20 20 --dtype f64 --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/tune/${v}_n$n.json 2> gpurun_out/tune/${v}_n$n.err
  done
done
echo done
