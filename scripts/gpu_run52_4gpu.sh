cd $GRAFT_REPO_ROOT
timeout -k 5 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t52_all.log 2>&1; echo "rc=$?" >> gpurun_out/t52_all.log
timeout -k 10 900 python bench.py > gpurun_out/b52_n1.log 2>&1; echo "rc=$?" >> gpurun_out/b52_n1.log
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552"
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29553"
timeout -k 10 900 $R2 bench.py --gpus 2 > gpurun_out/b52_n2.log 2>&1; echo "rc=$?" >> gpurun_out/b52_n2.log
timeout -k 10 900 $R4 bench.py --gpus 4 > gpurun_out/b52_n4.log 2>&1; echo "rc=$?" >> gpurun_out/b52_n4.log
timeout -k 10 900 $R4 bench.py --gpus 4 --stages 2 > gpurun_out/b52_n4_s2.log 2>&1; echo "rc=$?" >> gpurun_out/b52_n4_s2.log
timeout -k 10 900 $R4 bench.py --gpus 4 --workload failure > gpurun_out/b52_failure4.log 2>&1; echo "rc=$?" >> gpurun_out/b52_failure4.log
