#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 300 python scripts/tc_trace.py 30 30 30 > gpurun_out/tc_trace.txt 2>&1
echo done
