#!/bin/bash
# A/B of an env toggle on one box: alternating engine-headline runs (power-cap noise hits both)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
VAR=$1; A=$2; B=$3; R=${4:-2}; M=${MODEL:-C}
for i in $(seq 1 $R); do
  for v in $A $B; do
    env $VAR=$v timeout 400 python bench.py --workload engine --model $M --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; j=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$VAR=$v', round(j['value']), 'MHz', j['clocks']['sm_mhz'], 'gemm_ms', round(j['roofline']['gemm_ms_per_step'],1), 'frac', round(j['roofline']['frac'],3))"
  done
done
