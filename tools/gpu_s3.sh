#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
FDE_LIB_DEBUG=1 FDE_DEBUG2D=1 timeout 600 python tools/dbg_2d_paper.py > gpurun_out/dbg2d_v.log 2>&1; echo "dbg rc=$?" >> gpurun_out/dbg2d_v.log
grep -v "^  sign" gpurun_out/dbg2d_v.log | head -80
