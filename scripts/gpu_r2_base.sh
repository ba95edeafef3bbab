#!/bin/bash
# Round-2 baseline: GPU suite, bench line, full ncu capture of the C3 stage kernel.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out/r2base
O=gpurun_out/r2base
nvidia-smi > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu --durations=15 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench.json 2> $O/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_stage_kernel -s 5 -c 1 \
  -o $O/prof_tc_c3 python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/ncu_tc.log 2>&1
echo done
