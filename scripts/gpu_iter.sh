#!/bin/bash
# Iteration session: TC tests (short timeout), full GPU suite, bench, phase trace.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 150 python -m pytest tests/test_gpu_tc_stage.py -q -rA -x -s > gpurun_out/pytest_tc_stage.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc_stage.log
if grep -q "rc=0" gpurun_out/pytest_tc_stage.log; then
  timeout 600 python -m pytest tests -q -m gpu -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
  timeout 120 python scripts/tc_trace.py 30 30 30 > gpurun_out/tc_trace.txt 2>&1
fi
echo done
