cd $GRAFT_REPO_ROOT
export TORCH_NCCL_SHOW_EAGER_INIT_P2P_SERIALIZATION_WARNING=false
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591"
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29592"
for L in 1 2; do
timeout -k 10 900 $R4 bench.py --gpus 4 --workload engine --stages 2 --lanes $L > gpurun_out/b90_n4s2_l$L.log 2>&1; echo "rc=$?" >> gpurun_out/b90_n4s2_l$L.log
timeout -k 10 900 $R2 bench.py --gpus 2 --workload engine --lanes $L > gpurun_out/b90_n2_l$L.log 2>&1; echo "rc=$?" >> gpurun_out/b90_n2_l$L.log
done
timeout -k 10 900 $R4 bench.py --gpus 4 --workload engine --lanes 3 > gpurun_out/b90_n4_l3.log 2>&1; echo "rc=$?" >> gpurun_out/b90_n4_l3.log
