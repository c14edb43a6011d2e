cd $GRAFT_REPO_ROOT
export TORCH_NCCL_SHOW_EAGER_INIT_P2P_SERIALIZATION_WARNING=false
timeout -k 5 300 python scripts/ce_probe.py > gpurun_out/ce76.log 2>&1; echo "rc=$?" >> gpurun_out/ce76.log
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581"
timeout -k 10 900 $R4 bench.py --gpus 4 --workload engine > gpurun_out/b76_engine_n4.log 2>&1; echo "rc=$?" >> gpurun_out/b76_engine_n4.log
timeout -k 10 900 $R4 bench.py --gpus 4 --workload engine --stages 2 > gpurun_out/b76_engine_n4s2.log 2>&1; echo "rc=$?" >> gpurun_out/b76_engine_n4s2.log
timeout -k 10 900 python bench.py --workload engine > gpurun_out/b76_engine_n1.log 2>&1; echo "rc=$?" >> gpurun_out/b76_engine_n1.log
timeout -k 10 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches76.csv python bench.py --workload engine --steps 1 --warmup 3 > gpurun_out/ncu76.log 2>&1; echo "rc=$?" >> gpurun_out/ncu76.log
