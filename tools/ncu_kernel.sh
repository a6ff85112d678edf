#!/bin/bash
# usage: bash tools/ncu_kernel.sh <kernel-regex> <tag>  -- full ncu capture of one launch of the
# kernel in tools/prof_step.py (cfg3 fused steps), after a plain run of the same command.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python tools/prof_step.py 3 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s 1 -c 1 -o gpurun_out/prof_$2 python tools/prof_step.py 3 > gpurun_out/ncu_$2.log 2>&1
echo rc=$?
tail -2 gpurun_out/ncu_$2.log
