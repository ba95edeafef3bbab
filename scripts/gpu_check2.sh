#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --deselect tests/test_gpu_tc_stage.py -rf -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --path simt > gpurun_out/bench_simt.json 2> gpurun_out/bench_simt.err
timeout 300 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_tc_stage.py -q -x -k "selected_and_rhs and 1" > gpurun_out/sanitize_tc.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_tc.log
echo done
