#!/bin/bash
# Tensor-core path bring-up: probe, TC stage tests (short timeouts), full GPU suite, bench both paths.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gpu_tc05.py -x -q -rA -s > gpurun_out/pytest_tc05.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc05.log
timeout 180 python -m pytest tests/test_gpu_tc_stage.py -q -rA -s > gpurun_out/pytest_tc_stage.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc_stage.log
timeout 600 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --path simt > gpurun_out/bench_simt.json 2> gpurun_out/bench_simt.err
echo done
timeout 300 python scripts/tc_trace.py 30 30 30 > gpurun_out/tc_trace.txt 2>&1
