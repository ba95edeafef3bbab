#!/bin/bash
# Full GPU session: suite (auto path = tensor for N<=4 fp32), smoke, bench, launch list, TC trace, ncu full capture.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 120 python scripts/tc_trace.py 30 30 30 > gpurun_out/tc_trace.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_stage_kernel -s 3 -c 1 \
  -o gpurun_out/prof_tc python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
