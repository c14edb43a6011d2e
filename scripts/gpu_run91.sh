cd $GRAFT_REPO_ROOT
export TORCH_NCCL_SHOW_EAGER_INIT_P2P_SERIALIZATION_WARNING=false
timeout -k 5 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t91_all.log 2>&1; echo "rc=$?" >> gpurun_out/t91_all.log
timeout -k 5 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke91.log 2>&1; echo "rc=$?" >> gpurun_out/smoke91.log
timeout -k 10 1500 python bench.py > gpurun_out/b91_n1.log 2>&1; echo "rc=$?" >> gpurun_out/b91_n1.log
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29593"
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29594"
timeout -k 10 1500 $R2 bench.py --gpus 2 > gpurun_out/b91_n2.log 2>&1; echo "rc=$?" >> gpurun_out/b91_n2.log
timeout -k 10 1500 $R4 bench.py --gpus 4 > gpurun_out/b91_n4.log 2>&1; echo "rc=$?" >> gpurun_out/b91_n4.log
timeout -k 10 300 $R4 scripts/engine_multi_gpu_check.py 2 3 > gpurun_out/m91_n4s2.log 2>&1; echo "rc=$?" >> gpurun_out/m91_n4s2.log
