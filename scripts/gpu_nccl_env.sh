#!/bin/bash
# 4x1 engine line under different NCCL channel settings (do the p2p kernels steal SMs from the GEMMs?)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
i=0
for e in "X=1" "NCCL_MAX_NCHANNELS=1" "NCCL_MAX_NCHANNELS=4" "NCCL_P2P_USE_CUDA_MEMCPY=1" "NCCL_MAX_CTAS=2"; do
  i=$((i+1))
  env $e timeout 400 $TR --master-port 2954$i bench.py --gpus 4 --workload engine --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/nccl_$i.json 2> gpurun_out/nccl_$i.err
  python -c "
import json,sys; j=json.loads(open('gpurun_out/nccl_$i.json').read().strip().splitlines()[-1])
print('$e', round(j['value']), round(j['ms_per_step'],1), 'frac', round(j['roofline']['frac'],3), 'gemm_ms', round(j['roofline']['gemm_ms_per_step'],1), j['clocks']['sm_mhz'])" 2>&1 | tail -1
done
