#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
FDE_NVCC_FLAGS=-DFDE_FAKE_GJ python paper_1804_05522_b200/build.py > gpurun_out/s29_build.log 2>&1
FDE_LIB_DEBUG=1 FDE_TRACE_RUN=gpurun_out/run_trace.txt timeout 300 python tools/trace_run.py 16 > gpurun_out/s29.log 2>&1
grep "A phases\|span" gpurun_out/s29.log | head -3
