#!/bin/bash
# BASELINE configs[4] on N GPUs through the engine + C++ driver
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --workload failure > gpurun_out/failure_n$N.json 2> gpurun_out/failure_n$N.err
echo "failure rc=$?"; tail -c 1500 gpurun_out/failure_n$N.json; grep -v Warning gpurun_out/failure_n$N.err | tail -5
