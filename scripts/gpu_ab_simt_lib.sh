#!/bin/bash
# A/B of a SIMT/DMMA stage-kernel variant library against libdgm.so: parity (fp64 + fp32 SIMT tests) and
# stage time for fp64 (C3, 48k N=3, 6) and the fp32 SIMT orders (48k N=1, 2; C1 N=3 1,512 tets).
# usage: gpu_ab_simt_lib.sh libdgm_variant.so
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
V=$1; O=gpurun_out/ab_$V; mkdir -p $O
DGM_LIB=$PWD/paper_0901_1024_b200/$V timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py tests/test_gpu_unstructured.py -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -2 $O/tests.log
for rep in 1 2; do
  for lib in libdgm.so $V; do
    for cfg in "f64 4 55" "f64 3 20" "f64 6 20" "f32 1 20" "f32 2 20"; do
      set -- $cfg
      DGM_LIB=$PWD/paper_0901_1024_b200/$lib timeout 300 python bench.py --dtype $1 --order $2 --cells $3 $3 $3 --steps 10 --warmup 3 --extras none --no-cpu-baseline --e2e-steps 1 --dropin-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$1 N=$2 cells=$3', round(d['ms_per_step']/5*1e3,1), 'us/stage')"
    done
    DGM_LIB=$PWD/paper_0901_1024_b200/$lib timeout 300 python bench.py --order 3 --cells 6 6 7 --steps 200 --warmup 20 --extras none --no-cpu-baseline --e2e-steps 1 --dropin-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'f32 N=3 C1', round(d['ms_per_step']/5*1e3,2), 'us/stage')"
  done
done | tee $O/times.txt
