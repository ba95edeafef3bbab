#!/bin/bash
# A/B: default library vs the N=4 small-CTA experiment build.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out/ab
timeout 300 python -m pytest tests/test_gpu_tc_stage.py -q -x > gpurun_out/ab/tc_default.log 2>&1; echo "rc=$?" >> gpurun_out/ab/tc_default.log
DGM_LIB=$PWD/paper_0901_1024_b200/libdgm_late.so timeout 300 python -m pytest tests/test_gpu_tc_stage.py -q -x > gpurun_out/ab/tc_late.log 2>&1; echo "rc=$?" >> gpurun_out/ab/tc_small.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ab/bench_default.json 2> gpurun_out/ab/bench_default.err
DGM_LIB=$PWD/paper_0901_1024_b200/libdgm_late.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ab/bench_late.json 2> gpurun_out/ab/bench_late.err
echo done
