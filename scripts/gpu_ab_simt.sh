#!/bin/bash
# A/B of fp32 SIMT variant libraries at C2 N=1,2,3 (path simt) and C1
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
for lib in "$@"; do
  DGM_LIB=$PWD/paper_0901_1024_b200/$lib timeout 600 python -m pytest tests/test_gpu_tc_stage.py -x -q -k "simt" 2>&1 | tail -1 | sed "s/^/$lib parity: /"
  for n in 1 2 3; do
    DGM_LIB=$PWD/paper_0901_1024_b200/$lib timeout 300 python bench.py --path simt --order $n --cells 20 20 20 --steps 20 --warmup 3 --extras none --no-cpu-baseline --e2e-steps 1 --dropin-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'N=$n', round(d['ms_per_step']/5*1e3,1), 'us/stage')"
  done
done
