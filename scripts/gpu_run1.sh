set -x
cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/smi.txt 2>&1
timeout -k 10 600 python -m pytest tests -m gpu -q -k "not gemm" -p no:cacheprovider > gpurun_out/t_nongemm.log 2>&1; echo "rc=$?" >> gpurun_out/t_nongemm.log
timeout -k 10 400 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider > gpurun_out/t_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/t_gemm.log
timeout -k 10 300 python bench.py --steps 200 --warmup 5 > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
