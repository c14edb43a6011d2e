cd $GRAFT_REPO_ROOT
export TORCH_NCCL_SHOW_EAGER_INIT_P2P_SERIALIZATION_WARNING=false
timeout -k 5 600 python -m pytest tests/test_executor_gpu.py -x -q -p no:cacheprovider > gpurun_out/t57_exec.log 2>&1; echo "rc=$?" >> gpurun_out/t57_exec.log
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562"
timeout -k 10 300 $R4 scripts/engine_multi_gpu_check.py 2 3 > gpurun_out/m57_n4s2.log 2>&1; echo "rc=$?" >> gpurun_out/m57_n4s2.log
timeout -k 10 300 $R4 scripts/engine_multi_gpu_check.py 4 2 > gpurun_out/m57_n4.log 2>&1; echo "rc=$?" >> gpurun_out/m57_n4.log
timeout -k 10 900 $R4 bench.py --gpus 4 --workload engine --stages 2 > gpurun_out/b57_engine_n4s2.log 2>&1; echo "rc=$?" >> gpurun_out/b57_engine_n4s2.log
timeout -k 10 900 $R4 bench.py --gpus 4 --stages 2 --no-codec > gpurun_out/b57_train_n4s2.log 2>&1; echo "rc=$?" >> gpurun_out/b57_train_n4s2.log
