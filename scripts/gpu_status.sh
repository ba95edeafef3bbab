#!/bin/bash
# Status session: GPU tests (SIMT + TC separately, short timeouts), both bench paths, TC hang trace.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 600 python -m pytest tests -q -m gpu --deselect tests/test_gpu_tc_stage.py -rf > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 150 python -m pytest tests/test_gpu_tc_stage.py -q -rA -x > gpurun_out/pytest_tc_stage.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc_stage.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --path simt > gpurun_out/bench_simt.json 2> gpurun_out/bench_simt.err
timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --path tensor > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err
timeout 120 python scripts/tc_trace.py 10 10 10 > gpurun_out/tc_trace.txt 2>&1
echo done
