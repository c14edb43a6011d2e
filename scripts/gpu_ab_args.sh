#!/bin/bash
# engine headline with extra bench.py arguments vs the default, alternating (one box)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
run() {
  timeout 500 python bench.py --workload engine --steps 6 --warmup 3 --no-cpu-baseline $1 > gpurun_out/aba.json 2>/dev/null
  python -c "
import json; j=json.loads(open('gpurun_out/aba.json').read().strip().splitlines()[-1])
print('[$1]', round(j['value']), 'MHz', j['clocks']['sm_mhz'], 'frac', round(j['roofline']['frac'],3))"
}
for a in "$@"; do run ""; run "$a"; done
