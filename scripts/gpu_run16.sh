cd $GRAFT_REPO_ROOT
timeout -k 5 300 python -m pytest tests/test_gemm_gpu.py tests/test_stage_gpu.py tests/test_pipeline_gpu.py tests/test_attention_gpu.py tests/test_norm_gpu.py -q -p no:cacheprovider > gpurun_out/t16.log 2>&1; echo "rc=$?" >> gpurun_out/t16.log
timeout -k 5 300 python scripts/gemm_shapes.py --out gpurun_out/gemm_shapes16.json > gpurun_out/gemm_shapes16.log 2>&1
timeout -k 10 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b16_C.log 2>&1; echo "rc=$?" >> gpurun_out/b16_C.log
B="python bench.py --steps 1 --warmup 3 --microbatches 8 --no-cpu-baseline --no-codec"
timeout -k 10 600 $B > gpurun_out/b16_plain.log 2>&1 && \
timeout -k 10 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 12000 -c 5000 --csv --log-file gpurun_out/launches16.csv $B > gpurun_out/ncu_launch16.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_launch16.log
