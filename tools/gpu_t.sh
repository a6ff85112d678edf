#!/bin/bash
# quick check of the 2D step: parity tests (2D, split, rational Krylov) + wall time of cfg5 steps
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_2d.py tests/test_split2d.py tests/test_rk2d.py -q -m gpu -p no:cacheprovider > gpurun_out/t_2d.log 2>&1; echo "t rc=$?" >> gpurun_out/t_2d.log
tail -n 6 gpurun_out/t_2d.log
timeout 300 python tools/time_2d.py
timeout 300 python - <<'PY'
import sys; sys.path.insert(0, '.')
import torch, bench
print(bench.measure_cfg5(torch.device('cuda', 0), 1, 0))
PY
