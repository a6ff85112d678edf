#!/bin/bash
# k_run timing + 1D parity subset after a kernel change
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python tools/time_run.py 16 64 > gpurun_out/s32_time.log 2>&1; echo "time rc=$?" >> gpurun_out/s32_time.log
timeout 900 python -m pytest tests/test_parity_1d.py tests/test_parity_full.py tests/test_split1d.py -q -m gpu -x > gpurun_out/s32_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s32_pytest.log
cat gpurun_out/s32_time.log; tail -5 gpurun_out/s32_pytest.log
