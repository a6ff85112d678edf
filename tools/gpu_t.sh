#!/bin/bash
# ncu --set full of the 2D step's top kernels (cluster Gauss-Jordan inverse, tall-skinny GEMM) at cfg5
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python tools/prof_2d.py 3 > gpurun_out/plain2d.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gj_inv_cl -s 20 -c 2 -o gpurun_out/prof_2d python tools/prof_2d.py 3 > gpurun_out/ncu_2dfull.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu_2dfull.log
