#!/bin/bash
# balanced placement at N GPUs with env settings (VAR=VAL ... | none), alternating
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $N --master-port 29561"
for kv in "$@"; do
  env $kv timeout 600 $TR bench.py --gpus $N --workload engine --steps 20 --warmup 5 --no-cpu-baseline --placement balanced $EXTRA > gpurun_out/eb.json 2> gpurun_out/eb.err
  python -c "
import json; j=json.loads(open('gpurun_out/eb.json').read().strip().splitlines()[-1])
print('$kv', round(j['value']), 'MHz', j['clocks']['sm_mhz'], 'captures', j['engine']['graph_captures_in_timed_region_rank0'], 'e2e', round(j['e2e']['value']), j['e2e']['graph_captures_in_timed_region'])" || tail -3 gpurun_out/eb.err
done
