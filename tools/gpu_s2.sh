#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
FDE_LIB_DEBUG=1 timeout 600 python tools/dbg_2d_paper.py > gpurun_out/dbg2d.log 2>&1; echo "dbg rc=$?" >> gpurun_out/dbg2d.log
timeout 600 python tools/prof_2d.py 4 > gpurun_out/prof2d.log 2>&1; echo "prof2d rc=$?" >> gpurun_out/prof2d.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
tail -n 12 gpurun_out/dbg2d.log gpurun_out/prof2d.log; tail -c 600 gpurun_out/bench.err
