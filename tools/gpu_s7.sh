#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_rk2d.py tests/test_parity_2d.py tests/test_split2d.py -x > gpurun_out/trk.log 2>&1; echo "trk rc=$?" >> gpurun_out/trk.log
tail -n 30 gpurun_out/trk.log
