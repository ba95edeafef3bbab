#!/bin/bash
# A/B of fp64 variant libraries: parity (fp64 rhs all orders) + stage time at C3 and C2 N=3,5,6
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
O=gpurun_out/abf64; mkdir -p $O
LIBS=("$@")
for lib in "${LIBS[@]}"; do
  DGM_LIB=$PWD/paper_0901_1024_b200/$lib timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "dtype1" 2>&1 | tail -1 | sed "s/^/$lib parity: /"
done
for rep in 1 2; do
  for lib in "${LIBS[@]}"; do
    for cfg in "4 55" "3 20" "5 20" "6 20" "8 20" "9 20"; do
      set -- $cfg
      DGM_LIB=$PWD/paper_0901_1024_b200/$lib timeout 300 python bench.py --dtype f64 --order $1 --cells $2 $2 $2 --steps 10 --warmup 3 --extras none --no-cpu-baseline --e2e-steps 1 --dropin-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'N=$1', round(d['ms_per_step']/5*1e3,1), 'us/stage')"
    done
  done
done | tee $O/times.txt
