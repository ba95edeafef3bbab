#!/bin/bash
# Quick GPU session: GPU tests (with timeout) + bench.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tc05.py -x -q -rA -s > gpurun_out/pytest_tc05.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc05.log
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done
