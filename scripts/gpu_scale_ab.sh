#!/bin/bash
# A/B of attention env toggles on the N-GPU default bench (run under gpurun --gpus N)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $N --master-port 29541"
for rep in 1 2; do
for cfg in "SWARM_ATTN_LSE=1" "SWARM_ATTN_LSE=0" "SWARM_ATTN_BWD_FUSED=0"; do
  env $cfg timeout 600 $TR bench.py --gpus $N --workload engine --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sab.json 2>/dev/null
  python -c "
import json; j=json.loads(open('gpurun_out/sab.json').read().strip().splitlines()[-1])
print('$cfg', round(j['value']), 'MHz', j['clocks']['sm_mhz'])"
done
done
