#!/bin/bash
# NEXT-2 ladder up to the paper's N = 65536, cold-path timing.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python tools/paper2d.py gpurun_out/r02_paper2d.json > gpurun_out/paper2d.log 2>&1; echo "paper2d rc=$?" >> gpurun_out/paper2d.log
timeout 300 python tools/cold_path.py > gpurun_out/cold_path.log 2>&1; echo "cold rc=$?" >> gpurun_out/cold_path.log
tail -n 30 gpurun_out/paper2d.log; tail -n 15 gpurun_out/cold_path.log
