#!/bin/bash
# 16-producer-warp variant (libdgm_wide.so, N=5..9) vs the default kernels: parity + C2/C5 timing
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
O=gpurun_out/wide; mkdir -p $O
DGM_LIB=$PWD/paper_0901_1024_b200/libdgm_wide.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "all_orders and dtype0" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -2 $O/tests.log
for lib in libdgm.so libdgm_wide.so; do
  for n in 5 6 7 8 9; do
    DGM_LIB=$PWD/paper_0901_1024_b200/$lib timeout 300 python bench.py --order $n --cells 20 20 20 --steps 20 --warmup 3 --extras none --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', $n, round(d['ms_per_step']/5*1e3,1), 'us/stage')"
  done
done
