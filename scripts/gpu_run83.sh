cd $GRAFT_REPO_ROOT
export TORCH_NCCL_SHOW_EAGER_INIT_P2P_SERIALIZATION_WARNING=false
timeout -k 5 600 python -m pytest tests/test_stage_gpu.py tests/test_pipeline_gpu.py tests/test_executor_gpu.py -x -q -p no:cacheprovider > gpurun_out/t83.log 2>&1; echo "rc=$?" >> gpurun_out/t83.log
timeout -k 10 1500 python bench.py --model D --no-cpu-baseline --no-codec > gpurun_out/b83_D_n1.log 2>&1; echo "rc=$?" >> gpurun_out/b83_D_n1.log
