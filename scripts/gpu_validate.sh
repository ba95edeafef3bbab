#!/bin/bash
# Full validation of the committed library: GPU suite, smoke, default bench line, C2 order sweep,
# C4/C5/C3-fp64 lines, launch list and one ncu --set full capture of the tensor-core stage kernel.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
O=gpurun_out/val; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
for n in 2 3 4 5 6 7 8 9; do
  timeout 300 python bench.py --order $n --cells 20 20 20 --steps 10 --warmup 3 --e2e-steps 1 --dropin-steps 0 --no-cpu-baseline > $O/c2_n$n.json 2> $O/c2_n$n.err
done
timeout 600 python bench.py --dtype f64 --steps 10 --warmup 3 --e2e-steps 3 --no-cpu-baseline > $O/c3_f64.json 2> $O/c3_f64.err
timeout 1200 python bench.py --cells 110 110 110 --steps 10 --warmup 3 --e2e-steps 3 --no-cpu-baseline > $O/c4.json 2> $O/c4.err
timeout 900 python bench.py --order 6 --cells 70 70 70 --steps 10 --warmup 3 --e2e-steps 3 --no-cpu-baseline > $O/c5.json 2> $O/c5.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 12 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --dropin-steps 0 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_stage_kernel -s 3 -c 1 -o $O/prof_tc python bench.py --steps 1 --warmup 3 --e2e-steps 1 --dropin-steps 0 --no-cpu-baseline > $O/ncu_full.log 2>&1
echo done
