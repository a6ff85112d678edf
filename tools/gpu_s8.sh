#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_pgmres.py > gpurun_out/tpg.log 2>&1; echo "tpg rc=$?" >> gpurun_out/tpg.log
timeout 600 python tools/break_even.py > gpurun_out/break_even.json 2> gpurun_out/break_even.err; echo "be rc=$?" >> gpurun_out/break_even.err
tail -n 30 gpurun_out/tpg.log; cat gpurun_out/break_even.json; tail -5 gpurun_out/break_even.err
