#!/bin/bash
# C2 order sweep (48k tets, N=1..9, fp32), C3 fp64, launch list + ncu full capture of the TC kernel.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out/sweep
for n in 1 2 3 4 5 6 7 8 9; do
  timeout 300 python bench.py --order $n --cells 20 20 20 --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sweep/n$n.json 2> gpurun_out/sweep/n$n.err
done
for n in 1 2 3 4; do
  timeout 300 python bench.py --order $n --cells 20 20 20 --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline --path simt > gpurun_out/sweep/n${n}_simt.json 2> gpurun_out/sweep/n${n}_simt.err
done
timeout 300 python bench.py --dtype f64 --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sweep/c3_f64.json 2> gpurun_out/sweep/c3_f64.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 12 --csv --log-file gpurun_out/launches_v6.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_stage_kernel -s 3 -c 1 -o gpurun_out/prof_tc_v6 python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
