cd $GRAFT_REPO_ROOT
timeout -k 5 600 python -m pytest tests/test_attention_gpu.py tests/test_stage_gpu.py tests/test_pipeline_gpu.py -x -q -p no:cacheprovider > gpurun_out/t31.log 2>&1; echo "rc=$?" >> gpurun_out/t31.log
timeout -k 5 120 python scripts/attn_time.py > gpurun_out/attn31.log 2>&1
timeout -k 10 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b31_C.log 2>&1; echo "rc=$?" >> gpurun_out/b31_C.log
