cd $GRAFT_REPO_ROOT
timeout -k 5 600 python -m pytest tests/test_attention_gpu.py tests/test_gemm_gpu.py tests/test_stage_gpu.py -x -q -p no:cacheprovider > gpurun_out/t29.log 2>&1; echo "rc=$?" >> gpurun_out/t29.log
timeout -k 5 120 python scripts/attn_time.py > gpurun_out/attn29.log 2>&1
timeout -k 5 300 python scripts/gemm_shapes.py --out gpurun_out/gemm_shapes29.json > gpurun_out/gemm_shapes29.log 2>&1
timeout -k 10 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b29_C.log 2>&1; echo "rc=$?" >> gpurun_out/b29_C.log
