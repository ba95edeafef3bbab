#!/bin/bash
# Round 2: full GPU suite + sanitizers on tiny meshes.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
O=gpurun_out/r2tests; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -rf --durations=15 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -5 $O/pytest_gpu.log
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_small.py > $O/sanitize_$tool.log 2>&1
  echo "rc=$?" >> $O/sanitize_$tool.log
  tail -3 $O/sanitize_$tool.log
done
