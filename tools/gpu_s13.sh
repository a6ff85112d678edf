#!/bin/bash
# k_run phase breakdown (diagnostics library).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
FDE_LIB_DEBUG=1 FDE_TRACE_RUN=gpurun_out/run_trace.txt timeout 300 python tools/trace_run.py 16 > gpurun_out/s13.log 2>&1
echo "rc=$?" >> gpurun_out/s13.log
tail -n 30 gpurun_out/s13.log
