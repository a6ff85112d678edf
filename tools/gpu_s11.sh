#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -x tests/test_parity_1d.py tests/test_split1d.py tests/test_errors.py > gpurun_out/t1d.log 2>&1; echo "t1d rc=$?" >> gpurun_out/t1d.log
timeout 300 python bench.py --no-extra --no-cpu --no-e2e > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc=$?" >> gpurun_out/bench_q.err
FDE_LIB_DEBUG=1 timeout 300 python tools/task_profile.py 16 > gpurun_out/task_profile.json 2>&1
timeout 300 python bench.py --steps 16 --no-extra --no-e2e > gpurun_out/bench_cold.json 2>/dev/null
tail -n 4 gpurun_out/t1d.log; python -c "
import json;d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['other_variant'])"
tail -c 1500 gpurun_out/task_profile.json
