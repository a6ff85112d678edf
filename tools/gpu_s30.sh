#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for f in 0 1; do FDE_LIB_DEBUG=1 FDE_RUN_FUSE_AB=$f timeout 300 python tools/small_cfgs.py cfg3 n=16384 cfg2 >> gpurun_out/s30.log 2>&1; done
cat gpurun_out/s30.log
