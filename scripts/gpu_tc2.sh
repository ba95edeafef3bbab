#!/bin/bash
# v2 tensor kernel: quick check with the trap-on-hang library, probe (tf32 truncation), parity tests,
# then C3 timing of both tensor paths.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
O=gpurun_out/tc2; mkdir -p $O
DGM_LIB=$PWD/paper_0901_1024_b200/libdgm_trace.so timeout 120 python scripts/tc2_quick.py > $O/quick_trace.log 2>&1; echo "rc=$?" >> $O/quick_trace.log
cat $O/quick_trace.log | tail -12
grep -q "^rc=0" $O/quick_trace.log || exit 0
timeout 300 python -m pytest tests/test_gpu_tc05.py -q -s -k truncated > $O/probe.log 2>&1; echo "rc=$?" >> $O/probe.log
timeout 600 python -m pytest tests/test_gpu_tc2.py -x -q -s > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -3 $O/tests.log
if grep -q "^rc=0" $O/tests.log; then
  for p in tensor2 tensor; do
    timeout 300 python bench.py --steps 20 --warmup 3 --extras none --no-cpu-baseline --e2e-steps 2 --path $p > $O/bench_$p.json 2> $O/bench_$p.err
  done
fi
echo done
