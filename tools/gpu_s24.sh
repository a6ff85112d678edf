#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for sp in 0 1; do FDE_LIB_DEBUG=1 FDE_RUN_SPLIT=$sp timeout 300 python tools/small_cfgs.py n=8192 n=16384 n=32768 >> gpurun_out/s24.log 2>&1; done
cat gpurun_out/s24.log
