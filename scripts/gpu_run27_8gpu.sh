# 8 GPUs: configs[2] 4 stages x 2 peers, and configs[4] (failure + rebalancing, S=4 layout 3,1,2,2)
cd $GRAFT_REPO_ROOT
nvidia-smi topo -m > gpurun_out/topo27.txt 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29527"
timeout -k 10 900 $R bench.py --gpus 8 > gpurun_out/b27_n8.log 2>&1; echo "rc=$?" >> gpurun_out/b27_n8.log
timeout -k 10 900 $R bench.py --gpus 8 --workload failure > gpurun_out/b27_failure8.log 2>&1; echo "rc=$?" >> gpurun_out/b27_failure8.log
timeout -k 10 600 $R bench.py --gpus 8 --impl reference > gpurun_out/b27_ref8.log 2>&1; echo "rc=$?" >> gpurun_out/b27_ref8.log
