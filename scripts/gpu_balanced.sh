#!/bin/bash
# balanced placement (run under gpurun --gpus N): parity vs sequential replay, then engine A/B vs contiguous
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $N --master-port 29551"
[ -n "$SKIP_PARITY" ] || timeout 600 $TR scripts/engine_multi_gpu_check.py 4 2 1 balanced > gpurun_out/bal_parity_n$N.log 2>&1; echo "parity rc=$?"
grep -E "rel |ticks" gpurun_out/bal_parity_n$N.log | head -20
run() {
  timeout 600 $TR bench.py --gpus $N --workload engine --steps 10 --warmup 3 --no-cpu-baseline $1 > gpurun_out/bal.json 2> gpurun_out/bal.err
  python -c "
import json; j=json.loads(open('gpurun_out/bal.json').read().strip().splitlines()[-1])
print('[$1]', round(j['value']), 'MHz', j['clocks']['sm_mhz'], 'tick', round(j['run']['tick_cost']['share_of_step'], 4), 'captures', j['engine']['graph_captures_in_timed_region_rank0'], j['config']['parallelism'][:40])" || tail -5 gpurun_out/bal.err
}
for a in "$@"; do run "$a"; done
