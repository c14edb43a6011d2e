#!/bin/bash
# engine-path bench at N = 1 and N = $1 (default 2) GPUs
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
N=${1:-2}; M=${MODEL:-C}
timeout 600 python bench.py --workload engine --model $M --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/eng_n1_$M.json 2> gpurun_out/eng_n1_$M.err
echo "n1 rc=$?"; tail -c 600 gpurun_out/eng_n1_$M.json
if [ $N -gt 1 ]; then
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --workload engine --model $M --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/eng_n${N}_$M.json 2> gpurun_out/eng_n${N}_$M.err
echo "n$N rc=$?"; tail -c 600 gpurun_out/eng_n${N}_$M.json
fi
