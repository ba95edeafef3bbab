#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
for lib in "$@"; do
  DGM_LIB=$PWD/paper_0901_1024_b200/$lib timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "dtype1 and (7 or 8 or 9)" 2>&1 | tail -1 | sed "s/^/$lib parity: /"
  for n in 7 8 9; do
    DGM_LIB=$PWD/paper_0901_1024_b200/$lib timeout 300 python bench.py --dtype f64 --order $n --cells 20 20 20 --steps 5 --warmup 3 --extras none --no-cpu-baseline --e2e-steps 1 --dropin-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'N=$n', round(d['ms_per_step']/5*1e3,1), 'us/stage', round(d['roofline']['frac'],3))"
  done
done
