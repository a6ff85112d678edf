#!/bin/bash
# quick: k_run timing (cfg3) + task trace (diagnostics library)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 120 python tools/time_run.py 16 64 > gpurun_out/t_time.log 2>&1
FDE_LIB_DEBUG=1 timeout 120 python tools/trace_run.py 16 > gpurun_out/t_trace.log 2>&1
cat gpurun_out/t_time.log; grep -E "phases|units|span|mean" gpurun_out/t_trace.log | tail -24
