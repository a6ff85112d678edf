#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_parity_2d.py tests/test_parity_full.py -k "2d or cfg5 or residual or cache or paper" > gpurun_out/t2d.log 2>&1; echo "t2d rc=$?" >> gpurun_out/t2d.log
timeout 600 python tools/prof_2d.py 4 > gpurun_out/prof2d.log 2>&1; echo "prof2d rc=$?" >> gpurun_out/prof2d.log
FDE_LIB_DEBUG=1 FDE_DEBUG2D=1 timeout 600 python tools/dbg_2d_paper.py > gpurun_out/dbg2d_v.log 2>&1; echo "dbg rc=$?" >> gpurun_out/dbg2d_v.log
tail -n 30 gpurun_out/t2d.log; cat gpurun_out/prof2d.log; grep "^1e-11" gpurun_out/dbg2d_v.log
