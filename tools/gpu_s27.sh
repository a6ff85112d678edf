#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python tools/prof_cfg4.py 512 > gpurun_out/s27_cfg4.log 2>&1
timeout 1200 python -m pytest tests/test_parity_1d.py tests/test_parity_full.py tests/test_parity_2d.py -q -m gpu -x > gpurun_out/s27_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s27_pytest.log
cat gpurun_out/s27_cfg4.log; tail -3 gpurun_out/s27_pytest.log
