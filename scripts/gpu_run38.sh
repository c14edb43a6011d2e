cd $GRAFT_REPO_ROOT
timeout -k 5 600 python -m pytest tests/test_attention_gpu.py tests/test_stage_gpu.py -x -q -p no:cacheprovider > gpurun_out/t38.log 2>&1; echo "rc=$?" >> gpurun_out/t38.log
timeout -k 5 120 python scripts/attn_time.py > gpurun_out/attn38.log 2>&1
timeout -k 5 120 python scripts/attn_trace.py > gpurun_out/attn_trace38.log 2>&1
