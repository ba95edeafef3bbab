#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out/sweep
timeout 300 python -m pytest tests/test_gpu_tc_stage.py -q -rA -x -s > gpurun_out/pytest_tc_stage.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc_stage.log
if grep -q "rc=0" gpurun_out/pytest_tc_stage.log; then
  timeout 600 python -m pytest tests -q -m gpu -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
  for n in 9; do
    timeout 300 python bench.py --order $n --cells 20 20 20 --steps 10 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/sweep/n${n}_tc.json 2> gpurun_out/sweep/n${n}_tc.err
  done
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
fi
echo done
