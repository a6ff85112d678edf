#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
FDE_LIB_DEBUG=1 FDE_TRACE_LEVELS=1 timeout 300 python tools/prof_cfg4.py 512 > gpurun_out/s26.log 2>&1
grep "k_levels pass\|k_levels node\|refactor" gpurun_out/s26.log | head -6
grep "k_levels trace CTA 0" gpurun_out/s26.log | head -1 | cut -c1-1500
