#!/bin/bash
# Factor-once pipelined run (k_run inv mode): new tests against the bounds-checked library, then
# the product library, then the cfg1 / cfg4 timings of bench.py.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
SEL="factor_once or invariant or pipelined or cfg1 or chunk or cfg4"
FDE_LIB_DEBUG=1 timeout 600 python -m pytest tests/test_parity_1d.py tests/test_errors.py tests/test_parity_full.py -q -m gpu -p no:cacheprovider -k "$SEL" -x > gpurun_out/s36_dbg.log 2>&1; echo "dbg rc=$?" >> gpurun_out/s36_dbg.log
tail -n 5 gpurun_out/s36_dbg.log
timeout 600 python -m pytest tests/test_parity_1d.py tests/test_errors.py tests/test_parity_full.py -q -m gpu -p no:cacheprovider -k "$SEL" > gpurun_out/s36_prod.log 2>&1; echo "prod rc=$?" >> gpurun_out/s36_prod.log
tail -n 5 gpurun_out/s36_prod.log
timeout 600 python - > gpurun_out/s36_time.log 2>&1 <<'PY'
import json, torch, bench
dev = torch.device("cuda:0")
print(json.dumps(bench.measure_small(dev, "cfg1")), flush=True)
print(json.dumps(bench.measure_small(dev, "cfg2")), flush=True)
print(json.dumps(bench.measure_cfg4(dev, 1, 0)), flush=True)
PY
echo "time rc=$?" >> gpurun_out/s36_time.log
cat gpurun_out/s36_time.log | cut -c1-1500
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/s36_full.log 2>&1; echo "full rc=$?" >> gpurun_out/s36_full.log
tail -n 5 gpurun_out/s36_full.log
