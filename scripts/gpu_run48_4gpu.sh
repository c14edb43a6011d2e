cd $GRAFT_REPO_ROOT
timeout -k 5 600 python -m pytest tests/test_pipeline_gpu.py tests/test_stage_gpu.py -x -q -p no:cacheprovider > gpurun_out/t48.log 2>&1; echo "rc=$?" >> gpurun_out/t48.log
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29549"
timeout -k 10 900 $R4 bench.py --gpus 4 --stages 2 --dpu > gpurun_out/b48_n4_s2_dpu.log 2>&1; echo "rc=$?" >> gpurun_out/b48_n4_s2_dpu.log
timeout -k 10 900 $R4 bench.py --gpus 4 --stages 2 > gpurun_out/b48_n4_s2.log 2>&1; echo "rc=$?" >> gpurun_out/b48_n4_s2.log
timeout -k 10 900 $R4 bench.py --gpus 4 --dpu > gpurun_out/b48_n4_dpu.log 2>&1; echo "rc=$?" >> gpurun_out/b48_n4_dpu.log
timeout -k 10 900 python bench.py --dpu --no-cpu-baseline --no-codec > gpurun_out/b48_n1_dpu.log 2>&1; echo "rc=$?" >> gpurun_out/b48_n1_dpu.log
