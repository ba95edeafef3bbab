#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
timeout 150 python -m pytest tests/test_gpu_tc_stage.py -q -rA -x -s > gpurun_out/pytest_tc_stage.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc_stage.log
timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --path tensor > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --path simt > gpurun_out/bench_simt.json 2> gpurun_out/bench_simt.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 3 -c 6 --csv --log-file gpurun_out/launches_tc.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --path tensor > gpurun_out/ncu_tc.log 2>&1
echo done
