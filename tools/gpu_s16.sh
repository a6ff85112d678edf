#!/bin/bash
# cfg4 (batch 512) kept-factor path: plain run, then ncu --set full of the build and solve kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python tools/prof_cfg4.py 512 > gpurun_out/s16_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/s16_plain.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_levels|k_leaf$|k_leaf_apply|k_solve_level|k_solve_dots" -c 6 -o gpurun_out/prof_cfg4 python tools/prof_cfg4.py 512 > gpurun_out/s16_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/s16_ncu.log
cat gpurun_out/s16_plain.log; tail -3 gpurun_out/s16_ncu.log
