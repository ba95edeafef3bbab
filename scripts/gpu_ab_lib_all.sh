#!/bin/bash
# A/B of a variant library against libdgm.so at every tensor order: parity (fp32 / tensor tests) + stage
# time at C3 (N=4) and 48k tets for N=3, 5..9.  usage: gpu_ab_lib_all.sh libdgm_variant.so
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
V=$1; O=gpurun_out/ab_$V; mkdir -p $O
DGM_LIB=$PWD/paper_0901_1024_b200/$V timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc_stage.py tests/test_gpu_tc05.py -x -q -k "dtype0 or tensor or tc" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -2 $O/tests.log
for rep in 1 2; do
  for lib in libdgm.so $V; do
    for cfg in "4 55" "3 20" "5 20" "6 20" "7 20" "8 20" "9 20"; do
      set -- $cfg
      DGM_LIB=$PWD/paper_0901_1024_b200/$lib timeout 300 python bench.py --order $1 --cells $2 $2 $2 --steps 20 --warmup 3 --extras none --no-cpu-baseline --e2e-steps 1 --dropin-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'N=$1', round(d['ms_per_step']/5*1e3,1), 'us/stage')"
    done
  done
done | tee $O/times.txt
