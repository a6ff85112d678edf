#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -x tests/test_parity_1d.py tests/test_parity_full.py tests/test_errors.py tests/test_split1d.py tests/test_rank_study.py > gpurun_out/t1d.log 2>&1; echo "t1d rc=$?" >> gpurun_out/t1d.log
timeout 300 python bench.py --no-extra --no-cpu --no-e2e > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc=$?" >> gpurun_out/bench_q.err
FDE_LIB_DEBUG=1 timeout 300 python tools/task_profile.py 16 > gpurun_out/task_profile.json 2>&1
timeout 300 python tools/prof_cfg4.py > gpurun_out/prof_cfg4.log 2>&1
tail -n 4 gpurun_out/t1d.log; tail -c 300 gpurun_out/bench_q.json; cat gpurun_out/task_profile.json; tail -25 gpurun_out/prof_cfg4.log
