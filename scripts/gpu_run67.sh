cd $GRAFT_REPO_ROOT
export TORCH_NCCL_SHOW_EAGER_INIT_P2P_SERIALIZATION_WARNING=false
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571"
for tpp in 1 3; do
timeout -k 10 900 python bench.py --workload engine --trainers-per-peer $tpp > gpurun_out/b67_n1_t$tpp.log 2>&1; echo "rc=$?" >> gpurun_out/b67_n1_t$tpp.log
timeout -k 10 900 $R4 bench.py --gpus 4 --workload engine --trainers-per-peer $tpp > gpurun_out/b67_n4_t$tpp.log 2>&1; echo "rc=$?" >> gpurun_out/b67_n4_t$tpp.log
done
timeout -k 10 900 $R4 bench.py --gpus 4 --workload engine --stages 2 --trainers-per-peer 3 > gpurun_out/b67_n4s2_t3.log 2>&1; echo "rc=$?" >> gpurun_out/b67_n4s2_t3.log
