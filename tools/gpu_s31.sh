#!/bin/bash
# Baseline of the restored tree: cfg3 k_run timing, default bench, one ncu --set full k_run capture.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python tools/time_run.py 16 64 > gpurun_out/s31_time.log 2>&1
timeout 900 python bench.py > gpurun_out/s31_bench.json 2> gpurun_out/s31_bench.err; echo "bench rc=$?" >> gpurun_out/s31_bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_run -s 1 -c 1 -o gpurun_out/s31_prof python tools/time_run.py 16 > gpurun_out/s31_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/s31_ncu.log
cat gpurun_out/s31_time.log; tail -c 400 gpurun_out/s31_bench.err; tail -2 gpurun_out/s31_ncu.log
