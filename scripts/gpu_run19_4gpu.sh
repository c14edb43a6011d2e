# config E on 4 GPUs (2 stages: 3,1 -> rebalance -> fail -> rebalance) + 4-GPU default train
cd $GRAFT_REPO_ROOT
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514"
timeout -k 10 900 $R bench.py --gpus 4 --workload failure > gpurun_out/b19_failure.log 2>&1; echo "rc=$?" >> gpurun_out/b19_failure.log
timeout -k 10 900 $R bench.py --gpus 4 > gpurun_out/b19_n4.log 2>&1; echo "rc=$?" >> gpurun_out/b19_n4.log
