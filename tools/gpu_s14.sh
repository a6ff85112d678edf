#!/bin/bash
# Cold path (S1+S2) rewrite: compression tests + per-kernel times.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_1d.py tests/test_rank_study.py tests/test_errors.py -q -m gpu -x > gpurun_out/s14_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s14_pytest.log
timeout 300 python tools/cold_path.py > gpurun_out/s14_cold.log 2>&1; echo "cold rc=$?" >> gpurun_out/s14_cold.log
tail -n 5 gpurun_out/s14_pytest.log; cat gpurun_out/s14_cold.log
