cd $GRAFT_REPO_ROOT
timeout -k 5 600 python -m pytest tests/test_gemm_gpu.py tests/test_stage_gpu.py -x -q -p no:cacheprovider > gpurun_out/t82.log 2>&1; echo "rc=$?" >> gpurun_out/t82.log
timeout -k 5 300 python scripts/gemm_shapes.py --model D > gpurun_out/gs82_D.log 2>&1
timeout -k 5 300 python scripts/gemm_shapes.py --model C > gpurun_out/gs82_C.log 2>&1
