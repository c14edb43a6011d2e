cd $GRAFT_REPO_ROOT
export TORCH_NCCL_SHOW_EAGER_INIT_P2P_SERIALIZATION_WARNING=false
timeout -k 5 600 python -m pytest tests/test_executor_gpu.py tests/test_stage_gpu.py tests/test_norm_gpu.py -x -q -p no:cacheprovider > gpurun_out/t89.log 2>&1; echo "rc=$?" >> gpurun_out/t89.log
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29590"
timeout -k 10 300 $R4 scripts/engine_multi_gpu_check.py 2 3 2 > gpurun_out/m89_n4s2.log 2>&1; echo "rc=$?" >> gpurun_out/m89_n4s2.log
timeout -k 10 300 $R4 scripts/engine_multi_gpu_check.py 4 2 2 > gpurun_out/m89_n4.log 2>&1; echo "rc=$?" >> gpurun_out/m89_n4.log
for L in 1 2; do
timeout -k 10 900 $R4 bench.py --gpus 4 --workload engine --lanes $L > gpurun_out/b89_n4_l$L.log 2>&1; echo "rc=$?" >> gpurun_out/b89_n4_l$L.log
timeout -k 10 900 $R4 bench.py --gpus 4 --workload engine --model D --lanes $L > gpurun_out/b89_D_n4_l$L.log 2>&1; echo "rc=$?" >> gpurun_out/b89_D_n4_l$L.log
done
timeout -k 10 900 python bench.py --workload engine --lanes 2 > gpurun_out/b89_n1_l2.log 2>&1; echo "rc=$?" >> gpurun_out/b89_n1_l2.log
