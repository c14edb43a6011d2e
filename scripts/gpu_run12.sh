# first multi-GPU runs: 2 GPUs (2 stages/rank), S=1 x P=2 (all-reduce path), S=2 x P=1
cd $GRAFT_REPO_ROOT
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
timeout -k 10 900 $R bench.py --gpus 2 --steps 3 --warmup 3 --no-codec > gpurun_out/b12_n2.log 2>&1; echo "rc=$?" >> gpurun_out/b12_n2.log
timeout -k 10 600 $R bench.py --gpus 2 --steps 2 --warmup 3 --no-codec --stages 1 --microbatches 8 > gpurun_out/b12_n2_s1.log 2>&1; echo "rc=$?" >> gpurun_out/b12_n2_s1.log
timeout -k 10 600 $R bench.py --gpus 2 --steps 2 --warmup 3 --no-codec --stages 2 > gpurun_out/b12_n2_s2.log 2>&1; echo "rc=$?" >> gpurun_out/b12_n2_s2.log
