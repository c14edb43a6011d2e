#!/bin/bash
# tick cost on the peer streams (run under gpurun --gpus 4): 2 stages x 2 peers, with / without DPU
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for dpu in "" "--dpu"; do
  tag=eng22${dpu}
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 \
    bench.py --gpus $N --workload engine --stages 2 --steps 10 --warmup 3 --no-cpu-baseline $dpu > gpurun_out/$tag.json 2> gpurun_out/$tag.err
  echo "$tag rc=$?"
  python - "$tag" <<'PY'
import json, sys
j = json.loads(open(f"gpurun_out/{sys.argv[1]}.json").read().strip().splitlines()[-1])
print(sys.argv[1], round(j["value"]), j["ms_per_step"], j["run"].get("tick_cost"))
PY
done
