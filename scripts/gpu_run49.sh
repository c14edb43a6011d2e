cd $GRAFT_REPO_ROOT
timeout -k 5 600 python -m pytest tests/test_pipeline_gpu.py tests/test_stage_gpu.py -x -q -p no:cacheprovider > gpurun_out/t49.log 2>&1; echo "rc=$?" >> gpurun_out/t49.log
timeout -k 10 900 python bench.py --dpu --no-cpu-baseline --no-codec > gpurun_out/b49_n1_dpu.log 2>&1; echo "rc=$?" >> gpurun_out/b49_n1_dpu.log
