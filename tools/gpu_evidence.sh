#!/bin/bash
# Round-end style evidence: full GPU suite, smoke, default bench, ncu launch list of the bench,
# one ncu --set full capture of a k_run launch (K = 16).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/ev_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/ev_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ev_smoke.log
timeout 900 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo "bench rc=$?" >> gpurun_out/ev_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ev_ncu_list.log 2>&1; echo "ncu list rc=$?" >> gpurun_out/ev_ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_run -s 1 -c 1 -o gpurun_out/prof python tools/time_run.py 16 > gpurun_out/ev_ncu_full.log 2>&1; echo "ncu full rc=$?" >> gpurun_out/ev_ncu_full.log
tail -n 3 gpurun_out/ev_pytest.log; tail -n 2 gpurun_out/ev_smoke.log; tail -c 300 gpurun_out/ev_bench.err; tail -1 gpurun_out/ev_ncu_list.log; tail -1 gpurun_out/ev_ncu_full.log
