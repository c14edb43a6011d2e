# 4-GPU validation: default (4 stages x 1 peer) and 2 stages x 2 peers (p2p + stage-group all-reduce)
cd $GRAFT_REPO_ROOT
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513"
timeout -k 10 900 $R bench.py --gpus 4 --steps 4 --warmup 3 --no-codec > gpurun_out/b15_n4.log 2>&1; echo "rc=$?" >> gpurun_out/b15_n4.log
timeout -k 10 600 $R bench.py --gpus 4 --steps 3 --warmup 3 --no-codec --stages 2 > gpurun_out/b15_n4_s2.log 2>&1; echo "rc=$?" >> gpurun_out/b15_n4_s2.log
