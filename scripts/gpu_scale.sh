#!/bin/bash
# default bench at N = 2 and 4 (the driver's scaling protocol) + the 2x2 engine line with / without DPU
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 $N; do
  [ $n -gt $N ] && continue
  S=$(date +%s)
  timeout 900 $TR --nproc-per-node $n --master-port 2952$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/scale_n$n.json 2> gpurun_out/scale_n$n.err
  echo "default n=$n rc=$? secs=$(( $(date +%s) - S ))"
done
if [ $N -ge 4 ]; then
  for d in "" "--dpu"; do
    timeout 600 $TR --nproc-per-node 4 --master-port 29531 bench.py --gpus 4 --workload engine --stages 2 --steps 10 --warmup 3 --no-cpu-baseline $d > gpurun_out/eng22$d.json 2> gpurun_out/eng22$d.err
    echo "2x2 $d rc=$?"
  done
fi
