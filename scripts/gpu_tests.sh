#!/bin/bash
# GPU suite (optionally a subset: scripts/gpu_tests.sh tests/test_x.py) -> gpurun_out/tests/
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out/tests
timeout 1500 python -m pytest ${@:-tests} -x -q -m gpu -rf --durations=20 > gpurun_out/tests/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/tests/pytest_gpu.log
tail -3 gpurun_out/tests/pytest_gpu.log
