cd $GRAFT_REPO_ROOT
for d in 0 1 2 4 3 5 6 7; do SWARM_GEMM_DBG=$d CUDA_VISIBLE_DEVICES=0 timeout -k 5 120 python scripts/gemm_dbg.py >> gpurun_out/dbg13.log 2>&1; done
SWARM_GEMM_PAIR=0 CUDA_VISIBLE_DEVICES=0 timeout -k 5 120 python scripts/gemm_dbg.py >> gpurun_out/dbg13.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512"
timeout -k 10 600 $R bench.py --gpus 2 --steps 2 --warmup 3 --no-codec --stages 1 --microbatches 8 > gpurun_out/b13_n2_s1.log 2>&1; echo "rc=$?" >> gpurun_out/b13_n2_s1.log
timeout -k 10 900 $R bench.py --gpus 2 > gpurun_out/b13_n2_default.log 2>&1; echo "rc=$?" >> gpurun_out/b13_n2_default.log
