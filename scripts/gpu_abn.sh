#!/bin/bash
# A/B/n: default libdgm.so vs paper_0901_1024_b200/libdgm_<variant>.so for each variant argument,
# tc_stage parity for every variant, then benches interleaved twice (C3 default workload, or the
# bench arguments in $BENCH_ARGS).
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out/abn
for v in "$@"; do
  DGM_LIB=$PWD/paper_0901_1024_b200/libdgm_$v.so timeout 300 python -m pytest tests/test_gpu_tc_stage.py -q -x > gpurun_out/abn/tc_$v.log 2>&1
  echo "rc=$?" >> gpurun_out/abn/tc_$v.log
done
for rep in 1 2; do
  timeout 300 python bench.py ${BENCH_ARGS:---steps 20 --warmup 3} --no-cpu-baseline --e2e-steps 3 > gpurun_out/abn/bench_default_$rep.json 2> gpurun_out/abn/bench_default_$rep.err
  for v in "$@"; do
    DGM_LIB=$PWD/paper_0901_1024_b200/libdgm_$v.so timeout 300 python bench.py ${BENCH_ARGS:---steps 20 --warmup 3} --no-cpu-baseline --e2e-steps 3 > gpurun_out/abn/bench_${v}_$rep.json 2> gpurun_out/abn/bench_${v}_$rep.err
  done
done
echo done
