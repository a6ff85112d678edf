#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_1d.py tests/test_parity_full.py tests/test_split1d.py tests/test_errors.py -q -m gpu -x > gpurun_out/s25_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s25_pytest.log
timeout 300 python tools/small_cfgs.py cfg1 cfg2 n=16384 cfg3 > gpurun_out/s25_small.log 2>&1
tail -n 3 gpurun_out/s25_pytest.log; cat gpurun_out/s25_small.log
