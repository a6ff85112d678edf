#!/bin/bash
# bench through the watchdog thread (the multi-rank path of the extras) and the default bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
FDE_BENCH_WATCHDOG=1 timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_wd.json 2> gpurun_out/bench_wd.err; echo "rc=$?" >> gpurun_out/bench_wd.err
FDE_BENCH_WATCHDOG=1 FDE_BENCH_EXTRA_TIMEOUT=5 timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_wd2.json 2> gpurun_out/bench_wd2.err; echo "rc=$?" >> gpurun_out/bench_wd2.err
tail -c 600 gpurun_out/bench_wd.json; tail -3 gpurun_out/bench_wd.err; tail -c 400 gpurun_out/bench_wd2.json; tail -3 gpurun_out/bench_wd2.err
