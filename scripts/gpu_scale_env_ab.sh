#!/bin/bash
# env A/B on the N-GPU engine bench (run under gpurun --gpus N): baseline vs each VAR=VAL arg, alternating
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $N --master-port 29543"
run() {
  env "$@" timeout 600 $TR bench.py --gpus $N --workload engine --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sea.json 2>/dev/null
  python -c "
import json; j=json.loads(open('gpurun_out/sea.json').read().strip().splitlines()[-1])
print('$*', round(j['value']), 'MHz', j['clocks']['sm_mhz'])"
}
for kv in "$@"; do run SWARM_NONE=1; run $kv; done
