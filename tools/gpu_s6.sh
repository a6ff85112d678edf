#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_split1d.py tests/test_split2d.py tests/test_errors.py > gpurun_out/tsplit.log 2>&1; echo "tsplit rc=$?" >> gpurun_out/tsplit.log
timeout 300 python tools/split_timing.py > gpurun_out/split_timing.json 2> gpurun_out/split_timing.err; echo "rc=$?" >> gpurun_out/split_timing.err
tail -n 5 gpurun_out/tsplit.log; cat gpurun_out/split_timing.json; tail -3 gpurun_out/split_timing.err
