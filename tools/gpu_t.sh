#!/bin/bash
# quick 2D check: parity tests (2D, split, rational Krylov) + smoke
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_2d.py tests/test_split2d.py tests/test_rk2d.py -q -m gpu -p no:cacheprovider > gpurun_out/t_2d.log 2>&1; echo "t rc=$?" >> gpurun_out/t_2d.log
tail -n 4 gpurun_out/t_2d.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
