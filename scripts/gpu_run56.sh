cd $GRAFT_REPO_ROOT
timeout -k 5 600 python -m pytest tests/test_executor_gpu.py -x -q -p no:cacheprovider > gpurun_out/t56_exec.log 2>&1; echo "rc=$?" >> gpurun_out/t56_exec.log
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561"
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562"
timeout -k 10 300 $R4 scripts/engine_multi_gpu_check.py 4 2 > gpurun_out/m56_n4.log 2>&1; echo "rc=$?" >> gpurun_out/m56_n4.log
timeout -k 10 300 $R4 scripts/engine_multi_gpu_check.py 2 3 > gpurun_out/m56_n4s2.log 2>&1; echo "rc=$?" >> gpurun_out/m56_n4s2.log
timeout -k 10 300 $R2 scripts/engine_multi_gpu_check.py 4 1 > gpurun_out/m56_n2.log 2>&1; echo "rc=$?" >> gpurun_out/m56_n2.log
timeout -k 10 900 $R4 bench.py --gpus 4 --workload engine > gpurun_out/b56_engine_n4.log 2>&1; echo "rc=$?" >> gpurun_out/b56_engine_n4.log
timeout -k 10 900 $R4 bench.py --gpus 4 > gpurun_out/b56_train_n4.log 2>&1; echo "rc=$?" >> gpurun_out/b56_train_n4.log
timeout -k 10 900 $R2 bench.py --gpus 2 --workload engine > gpurun_out/b56_engine_n2.log 2>&1; echo "rc=$?" >> gpurun_out/b56_engine_n2.log
