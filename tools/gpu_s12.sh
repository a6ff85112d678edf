#!/bin/bash
# Validate FDE_HOST_PTRS run + bench e2e path.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_1d.py -q -m gpu -x > gpurun_out/s12_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s12_pytest.log
timeout 600 python bench.py > gpurun_out/s12_bench.json 2> gpurun_out/s12_bench.err; echo "bench rc=$?" >> gpurun_out/s12_bench.err
tail -n 3 gpurun_out/s12_pytest.log; tail -c 300 gpurun_out/s12_bench.err; head -c 3000 gpurun_out/s12_bench.json
