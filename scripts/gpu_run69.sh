cd $GRAFT_REPO_ROOT
export TORCH_NCCL_SHOW_EAGER_INIT_P2P_SERIALIZATION_WARNING=false
timeout -k 5 600 python -m pytest tests/test_executor_gpu.py -x -q -p no:cacheprovider > gpurun_out/t69.log 2>&1; echo "rc=$?" >> gpurun_out/t69.log
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29574"
timeout -k 10 300 $R4 scripts/engine_multi_gpu_check.py 2 3 > gpurun_out/m69_n4s2.log 2>&1; echo "rc=$?" >> gpurun_out/m69_n4s2.log
timeout -k 10 900 python bench.py --workload engine > gpurun_out/b69_n1.log 2>&1; echo "rc=$?" >> gpurun_out/b69_n1.log
timeout -k 10 900 $R4 bench.py --gpus 4 --workload engine > gpurun_out/b69_n4.log 2>&1; echo "rc=$?" >> gpurun_out/b69_n4.log
timeout -k 10 900 $R4 bench.py --gpus 4 --workload engine --stages 2 --trainers-per-peer 4 > gpurun_out/b69_n4s2t4.log 2>&1; echo "rc=$?" >> gpurun_out/b69_n4s2t4.log
