#!/bin/bash
# Round 2: full bench line (all config rows), reference arm, launch list of the default bench command,
# ncu --set full of every config's stage kernel on an LSRK stage with a != 0 (launch 7 = stage 1 of the
# second warm-up step), summarised on the box; reports deleted except C3 (gpurun_out < 64 MiB).
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
O=gpurun_out/r2bench; mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c3.csv \
  python bench.py --steps 2 --warmup 3 --extras none --no-cpu-baseline --e2e-steps 1 --dropin-steps 0 > $O/launch_run.log 2>&1
cap() {  # name order "cells" dtype keep
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 6 -c 1 -o $O/prof_$1 \
    python bench.py --order $2 --cells $3 --dtype $4 --steps 1 --warmup 3 --extras none --no-cpu-baseline \
    --e2e-steps 1 --dropin-steps 0 > $O/ncu_$1.log 2>&1
  ncu -i $O/prof_$1.ncu-rep --page raw --csv > $O/raw_$1.csv 2>/dev/null
  python scripts/ncu_summary.py $O/raw_$1.csv $O/ncu_$1_summary.csv
  rm -f $O/raw_$1.csv
  [ "$5" = keep ] || rm -f $O/prof_$1.ncu-rep
}
cap c3 4 "55 55 55" f32 keep
cap c3f64 4 "55 55 55" f64
cap c5 6 "70 70 70" f32
for n in 1 2 3 4 5 6 7 8 9; do cap c2n$n $n "20 20 20" f32; done
cap c1 3 "6 6 7" f32
cap c4 4 "110 110 110" f32
du -sh $O
echo done
