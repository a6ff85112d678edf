#!/bin/bash
# k_run parity (1D) + phase trace.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_1d.py tests/test_parity_full.py tests/test_split1d.py -q -m gpu -x > gpurun_out/s17_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s17_pytest.log
FDE_LIB_DEBUG=1 FDE_TRACE_RUN=gpurun_out/run_trace.txt timeout 300 python tools/trace_run.py 16 > gpurun_out/s17_trace.log 2>&1
timeout 300 python tools/time_run.py > gpurun_out/s17_time.log 2>&1
tail -n 3 gpurun_out/s17_pytest.log; grep "phases\|units\|span\|A leaf\|B proj\|B' rhs\|L8\|L7" gpurun_out/s17_trace.log | head -14; tail -5 gpurun_out/s17_time.log
