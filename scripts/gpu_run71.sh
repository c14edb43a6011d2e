cd $GRAFT_REPO_ROOT
export TORCH_NCCL_SHOW_EAGER_INIT_P2P_SERIALIZATION_WARNING=false
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29577"
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29578"
timeout -k 10 300 $R4 scripts/engine_multi_gpu_check.py 2 3 > gpurun_out/m71_n4s2.log 2>&1; echo "rc=$?" >> gpurun_out/m71_n4s2.log
timeout -k 10 300 $R2 scripts/engine_multi_gpu_check.py 4 2 > gpurun_out/m71_n2.log 2>&1; echo "rc=$?" >> gpurun_out/m71_n2.log
timeout -k 10 900 $R4 bench.py --gpus 4 --workload engine --stages 2 --trainers-per-peer 4 > gpurun_out/b71_n4s2t4.log 2>&1; echo "rc=$?" >> gpurun_out/b71_n4s2t4.log
timeout -k 10 900 $R4 bench.py --gpus 4 --workload engine --stages 2 > gpurun_out/b71_n4s2.log 2>&1; echo "rc=$?" >> gpurun_out/b71_n4s2.log
timeout -k 10 900 $R4 bench.py --gpus 4 --workload engine > gpurun_out/b71_n4.log 2>&1; echo "rc=$?" >> gpurun_out/b71_n4.log
timeout -k 10 900 $R2 bench.py --gpus 2 --workload engine > gpurun_out/b71_n2.log 2>&1; echo "rc=$?" >> gpurun_out/b71_n2.log
