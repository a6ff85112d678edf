#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
FDE_LIB_DEBUG=1 FDE_TRACE_RUN=gpurun_out/run_trace.txt timeout 300 python tools/trace_run.py 16 > gpurun_out/s22_trace.log 2>&1; echo "trace rc=$?" >> gpurun_out/s22_trace.log
timeout 300 python tools/time_run.py 16 32 64 > gpurun_out/s22_time.log 2>&1
timeout 900 python -m pytest tests/test_parity_1d.py -q -m gpu -x -k "run or pipelined" > gpurun_out/s22_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s22_pytest.log
grep "phases\|units\|span\|rc=" gpurun_out/s22_trace.log | head -9; grep -A30 "span" gpurun_out/s22_trace.log | grep "^  " | head -30; tail -4 gpurun_out/s22_time.log; tail -3 gpurun_out/s22_pytest.log
