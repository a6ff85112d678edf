#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for sp in 0 1; do FDE_LIB_DEBUG=1 FDE_RUN_SPLIT=$sp timeout 300 python tools/small_cfgs.py >> gpurun_out/s23.log 2>&1; done
FDE_LIB_DEBUG=1 FDE_RUN_SPLIT=1 FDE_TRACE_RUN=gpurun_out/run_trace.txt timeout 300 python tools/trace_run.py 16 > gpurun_out/s23_trace.log 2>&1
cat gpurun_out/s23.log; grep -A40 "span" gpurun_out/s23_trace.log | head -30
