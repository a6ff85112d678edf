#!/bin/bash
# Evidence for the 2D step (cfg5) and the cold path (S1 + S2): per-kernel time table, ncu launch
# list of a 3-step cfg5 run, ncu --set full of k_pchol / k_eig (cfg3 compression).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python tools/prof_2d.py 16 > gpurun_out/prof2d.log 2>&1; echo "prof2d rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_2d.csv python tools/prof_2d.py 3 > gpurun_out/ncu_2d.log 2>&1; echo "ncu 2d list rc=$?"
timeout 300 python tools/cold_path.py > gpurun_out/cold_path.log 2>&1; echo "cold rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_pchol|k_eig' -c 4 -o gpurun_out/prof_cold python tools/cold_path.py > gpurun_out/ncu_cold.log 2>&1; echo "ncu cold rc=$?"
tail -n 40 gpurun_out/prof2d.log
