#!/bin/bash
# A/B: L2 prefetch of X^(m-1) by TMA tensor prefetch at the start of B' (abtmp/xpf.so vs base)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python tools/ab_libs.py abtmp/base.so abtmp/xpf.so abtmp/base.so abtmp/xpf.so > gpurun_out/s39_ab.log 2>&1; echo "ab rc=$?" >> gpurun_out/s39_ab.log
cat gpurun_out/s39_ab.log
timeout 900 python -m pytest tests/test_parity_1d.py -q -m gpu -p no:cacheprovider -x > gpurun_out/s39_t.log 2>&1; echo "t rc=$?" >> gpurun_out/s39_t.log
tail -n 3 gpurun_out/s39_t.log
