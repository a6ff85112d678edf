#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
FDE_LIB_DEBUG=1 FDE_TRACE_RUN=gpurun_out/run_trace.txt timeout 300 python tools/trace_run.py 16 > gpurun_out/s18_trace.log 2>&1
timeout 300 python tools/time_run.py 16 32 64 > gpurun_out/s18_time.log 2>&1
grep "phases\|units\|span" gpurun_out/s18_trace.log | head -7; tail -4 gpurun_out/s18_time.log
