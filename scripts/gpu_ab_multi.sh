#!/bin/bash
# several env A/Bs of the engine headline on one box (baseline run between each): VAR=VAL pairs as args
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
run() {
  env "$@" timeout 400 python bench.py --workload engine --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/abm.json 2>/dev/null
  python -c "
import json; j=json.loads(open('gpurun_out/abm.json').read().strip().splitlines()[-1])
print('$*', round(j['value']), 'MHz', j['clocks']['sm_mhz'], 'frac', round(j['roofline']['frac'],3))"
}
for kv in "$@"; do run SWARM_NONE=1; run $kv; done
run SWARM_NONE=1
