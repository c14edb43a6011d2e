# N=2 and N=4 of configs[2], configs[4] on 4 GPUs, the reference arm under torchrun
cd $GRAFT_REPO_ROOT
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29537"
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29538"
timeout -k 10 900 $R2 bench.py --gpus 2 > gpurun_out/b37_n2.log 2>&1; echo "rc=$?" >> gpurun_out/b37_n2.log
timeout -k 10 900 $R4 bench.py --gpus 4 > gpurun_out/b37_n4.log 2>&1; echo "rc=$?" >> gpurun_out/b37_n4.log
timeout -k 10 900 $R4 bench.py --gpus 4 --workload failure > gpurun_out/b37_failure4.log 2>&1; echo "rc=$?" >> gpurun_out/b37_failure4.log
timeout -k 10 900 $R4 bench.py --gpus 4 --impl reference > gpurun_out/b37_ref4.log 2>&1; echo "rc=$?" >> gpurun_out/b37_ref4.log
timeout -k 10 900 $R4 bench.py --gpus 4 --stages 2 > gpurun_out/b37_n4_s2.log 2>&1; echo "rc=$?" >> gpurun_out/b37_n4_s2.log
