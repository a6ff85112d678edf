#!/bin/bash
# Round-end check on the final tree: full GPU suite, smoke, default bench (no profiler).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/fin_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fin_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fin_smoke.log
timeout 900 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; echo "bench rc=$?" >> gpurun_out/fin_bench.err
tail -n 3 gpurun_out/fin_pytest.log; tail -n 2 gpurun_out/fin_smoke.log; tail -c 200 gpurun_out/fin_bench.err
