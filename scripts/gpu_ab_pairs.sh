#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py tests/test_gpu_unstructured.py tests/test_gpu_tc_stage.py -q 2>&1 | tail -1
for rep in 1 2; do
for lib in libdgm.so libdgm_nopairs.so; do
  for cfg in "f64 4 55" "f64 3 20" "f64 6 20" "f32 1 20" "f32 2 20"; do
    set -- $cfg
    DGM_LIB=$PWD/paper_0901_1024_b200/$lib timeout 300 python bench.py --dtype $1 --order $2 --cells $3 $3 $3 --steps 10 --warmup 3 --extras none --no-cpu-baseline --e2e-steps 1 --dropin-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$1 N=$2', round(d['ms_per_step']/5*1e3,1), 'us/stage')"
  done
done
done
