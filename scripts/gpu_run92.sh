cd $GRAFT_REPO_ROOT
export TORCH_NCCL_SHOW_EAGER_INIT_P2P_SERIALIZATION_WARNING=false
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29595"
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29596"
timeout -k 10 1500 $R2 bench.py --gpus 2 --model D --workload engine > gpurun_out/b92_D_n2.log 2>&1; echo "rc=$?" >> gpurun_out/b92_D_n2.log
timeout -k 10 1500 $R4 bench.py --gpus 4 --model D --workload engine --stages 2 > gpurun_out/b92_D_n4s2.log 2>&1; echo "rc=$?" >> gpurun_out/b92_D_n4s2.log
