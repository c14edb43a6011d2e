cd $GRAFT_REPO_ROOT
timeout -k 5 600 python -m pytest tests/test_attention_gpu.py tests/test_stage_gpu.py tests/test_pipeline_gpu.py -x -q -p no:cacheprovider > gpurun_out/t32.log 2>&1; echo "rc=$?" >> gpurun_out/t32.log
timeout -k 5 300 ncu --set full --import-source on --clock-control none -k regex:k_attn_chunks -c 2 -o gpurun_out/ncu_attn32 python scripts/attn_time.py > gpurun_out/ncu_attn32.log 2>&1
