cd $GRAFT_REPO_ROOT
timeout -k 5 120 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider -k "test_gemm_bf16 and 256-512-512" > gpurun_out/t8_small.log 2>&1; echo "rc=$?" >> gpurun_out/t8_small.log
if grep -q "rc=0" gpurun_out/t8_small.log; then
timeout -k 5 300 python -m pytest tests/test_gemm_gpu.py -q -p no:cacheprovider > gpurun_out/t8_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/t8_gemm.log
timeout -k 5 300 python scripts/gemm_shapes.py --out gpurun_out/gemm_shapes8_pair.json > gpurun_out/gemm_shapes8_pair.log 2>&1
SWARM_GEMM_PAIR=0 timeout -k 5 300 python scripts/gemm_shapes.py > gpurun_out/gemm_shapes8_single.log 2>&1
fi
