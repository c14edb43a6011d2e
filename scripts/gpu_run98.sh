cd $GRAFT_REPO_ROOT
export TORCH_NCCL_SHOW_EAGER_INIT_P2P_SERIALIZATION_WARNING=false
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29599"
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29600"
timeout -k 10 900 $R4 bench.py --gpus 4 --workload engine --trainers-per-peer 3 > gpurun_out/b98_n4_t3.log 2>&1; echo "rc=$?" >> gpurun_out/b98_n4_t3.log
timeout -k 10 900 $R2 bench.py --gpus 2 --workload engine --trainers-per-peer 3 > gpurun_out/b98_n2_t3.log 2>&1; echo "rc=$?" >> gpurun_out/b98_n2_t3.log
