#!/bin/bash
# Copy a gpu_r2_bench.sh / gpu_r2_tests.sh run (gpurun_out/r2bench, r2tests) into profiles/r02 and refresh
# profiles/ncu_summary.json (the traffic table bench.py reads).
cd "$(dirname "$0")/.."
S=gpurun_out/r2bench; T=gpurun_out/r2tests; D=profiles/r02/ncu
if [ -f $S/bench.json ]; then
  tail -1 $S/bench.json > profiles/r02/bench_r02_full.json
  cp $S/bench_ref.json profiles/r02/bench_ref_r02.json
  cp $S/ncu_*_summary.csv $S/launches_c3.csv $D/
  python scripts/update_ncu_summary.py "tc_stage_kernel<4>/f32@998250=$D/ncu_c3_summary.csv" \
    "stage_kernel<4>/f64@998250=$D/ncu_c3f64_summary.csv" "tc_stage_kernel<6>/f32@2058000=$D/ncu_c5_summary.csv" \
    "stage_kernel<1>/f32@48000=$D/ncu_c2n1_summary.csv" "stage_kernel<2>/f32@48000=$D/ncu_c2n2_summary.csv" \
    "tc_stage_kernel<3>/f32@48000=$D/ncu_c2n3_summary.csv" "tc_stage_kernel<4>/f32@48000=$D/ncu_c2n4_summary.csv" \
    "tc_stage_kernel<5>/f32@48000=$D/ncu_c2n5_summary.csv" "tc_stage_kernel<6>/f32@48000=$D/ncu_c2n6_summary.csv" \
    "tc_stage_kernel<7>/f32@48000=$D/ncu_c2n7_summary.csv" "tc_stage_kernel<8>/f32@48000=$D/ncu_c2n8_summary.csv" \
    "tc_stage_kernel<9>/f32@48000=$D/ncu_c2n9_summary.csv" \
    "stage_kernel<3>/f32@1512=$D/ncu_c1_summary.csv" "tc_stage_kernel<4>/f32@7986000=$D/ncu_c4_summary.csv"
fi
if [ -f $T/pytest_gpu.log ]; then
  cp $T/pytest_gpu.log profiles/r02/pytest_gpu_r2.log
  for t in memcheck synccheck racecheck; do [ -f $T/sanitize_$t.log ] && cp $T/sanitize_$t.log profiles/r02/sanitize/; done
fi
git status --short profiles
