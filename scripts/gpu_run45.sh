cd $GRAFT_REPO_ROOT
timeout -k 5 600 python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider > gpurun_out/t45.log 2>&1; echo "rc=$?" >> gpurun_out/t45.log
timeout -k 5 300 python scripts/gemm_shapes.py --model D --out gpurun_out/gemm_shapes45_D.json > gpurun_out/gemm_shapes45_D.log 2>&1
SWARM_GEMM_STREAMK=0 timeout -k 10 900 python bench.py --model D --steps 3 --warmup 3 --no-codec --no-cpu-baseline > gpurun_out/b45_D_nosk.log 2>&1; echo "rc=$?" >> gpurun_out/b45_D_nosk.log
