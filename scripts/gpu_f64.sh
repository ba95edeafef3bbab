#!/bin/bash
# fp64 stage kernel (DMMA P2): parity tests, then C3 fp64 + C2 fp64 order timing.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
O=gpurun_out/f64; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py tests/test_gpu_api.py tests/test_gpu_unstructured.py -x -q -rf > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -3 $O/tests.log
if grep -q "^rc=0" $O/tests.log; then
  timeout 600 python bench.py --dtype f64 --steps 10 --warmup 3 --extras none --no-cpu-baseline --e2e-steps 1 --dropin-steps 0 > $O/bench_c3_f64.json 2> $O/bench_c3_f64.err
  for n in 1 2 3 5 6; do
    timeout 300 python bench.py --dtype f64 --order $n --cells 20 20 20 --steps 10 --warmup 3 --extras none --no-cpu-baseline --e2e-steps 1 --dropin-steps 0 > $O/bench_c2_f64_n$n.json 2>> $O/bench_c2.err
  done
fi
echo done
