#!/bin/bash
# A/B: first-stripe cp.async prefetch during the LU + coop-stripe SMSP balance (abtmp/new.so vs base)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python tools/ab_libs.py abtmp/base.so abtmp/pc.so abtmp/p.so abtmp/c.so abtmp/base.so abtmp/pc.so abtmp/p.so abtmp/c.so > gpurun_out/s38_ab.log 2>&1; echo "ab rc=$?" >> gpurun_out/s38_ab.log
cat gpurun_out/s38_ab.log
timeout 900 python -m pytest tests/test_parity_1d.py -q -m gpu -p no:cacheprovider -x > gpurun_out/s38_t.log 2>&1; echo "t rc=$?" >> gpurun_out/s38_t.log
tail -n 3 gpurun_out/s38_t.log
