#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_split2d.py tests/test_parity_2d.py tests/test_parity_full.py -k "2d or cfg5 or residual or cache or paper or split" > gpurun_out/t2d.log 2>&1; echo "t2d rc=$?" >> gpurun_out/t2d.log
timeout 600 python tools/prof_2d.py 4 > gpurun_out/prof2d.log 2>&1; echo "prof2d rc=$?" >> gpurun_out/prof2d.log
tail -n 5 gpurun_out/t2d.log; head -14 gpurun_out/prof2d.log
