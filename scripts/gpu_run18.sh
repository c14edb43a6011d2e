cd $GRAFT_REPO_ROOT
timeout -k 5 300 python -m pytest tests/test_attention_gpu.py tests/test_stage_gpu.py -q -p no:cacheprovider > gpurun_out/t18.log 2>&1; echo "rc=$?" >> gpurun_out/t18.log
cp scripts/attn_time.py /tmp/ 2>/dev/null; timeout -k 5 120 python scripts/attn_time.py > gpurun_out/attn18.log 2>&1
timeout -k 10 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b18_C.log 2>&1; echo "rc=$?" >> gpurun_out/b18_C.log
