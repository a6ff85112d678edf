#!/bin/bash
# one ncu --set full capture (with source) of a K=16 k_run launch; tag = $1
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 120 python tools/time_run.py 16 > gpurun_out/ncu_plain_$1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_run -s 1 -c 1 -o gpurun_out/prof_$1 python tools/time_run.py 16 > gpurun_out/ncu_$1.log 2>&1
echo rc=$?; tail -2 gpurun_out/ncu_$1.log
