#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck on tiny meshes (scripts/sanitize_small.py)
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
O=gpurun_out/sanitize; mkdir -p $O
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_small.py "$@" > $O/$tool.log 2>&1
  echo "rc=$?" >> $O/$tool.log
  tail -3 $O/$tool.log
done
