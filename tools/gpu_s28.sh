#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python tools/cold_path.py > gpurun_out/s28_cold.log 2>&1
timeout 1500 python -m pytest tests/test_parity_1d.py tests/test_rank_study.py tests/test_parity_2d.py -q -m gpu -x > gpurun_out/s28_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s28_pytest.log
cat gpurun_out/s28_cold.log; tail -3 gpurun_out/s28_pytest.log
