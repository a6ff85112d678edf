#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_1d.py tests/test_parity_full.py tests/test_split1d.py tests/test_errors.py -q -m gpu -x > gpurun_out/s19_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s19_pytest.log
tail -n 3 gpurun_out/s19_pytest.log
