#!/bin/bash
# quick check: host-pointer tests + a short bench (e2e through FDE_HOST_PTRS)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_1d.py -q -m gpu -p no:cacheprovider -k "host_pointer or chunk" > gpurun_out/t_host.log 2>&1; echo "t rc=$?" >> gpurun_out/t_host.log
tail -n 15 gpurun_out/t_host.log
for i in 1 2; do timeout 600 python bench.py --no-extra --no-cpu > gpurun_out/bench_e2e_$i.json 2> gpurun_out/bench_e2e_$i.err; echo "bench rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/bench_e2e_$i.json').read().strip().splitlines()[-1]);print(d['value'],d['e2e']['value'],d['steps'])"; done
