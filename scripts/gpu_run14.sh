cd $GRAFT_REPO_ROOT
timeout -k 5 90 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider -k "test_gemm_bf16 and 2048-2048-2048" > gpurun_out/t14_small.log 2>&1; echo "rc=$?" >> gpurun_out/t14_small.log
if grep -q "rc=0" gpurun_out/t14_small.log; then
timeout -k 5 300 python -m pytest tests/test_gemm_gpu.py tests/test_stage_gpu.py tests/test_pipeline_gpu.py -q -p no:cacheprovider > gpurun_out/t14.log 2>&1; echo "rc=$?" >> gpurun_out/t14.log
timeout -k 5 120 python scripts/gemm_dbg.py > gpurun_out/dbg14.log 2>&1
SWARM_GEMM_MCAST=0 timeout -k 5 120 python scripts/gemm_dbg.py >> gpurun_out/dbg14.log 2>&1
timeout -k 5 300 python scripts/gemm_shapes.py --out gpurun_out/gemm_shapes14.json > gpurun_out/gemm_shapes14.log 2>&1
timeout -k 10 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b14_C.log 2>&1; echo "rc=$?" >> gpurun_out/b14_C.log
fi
