cd $GRAFT_REPO_ROOT
timeout -k 5 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t44_all.log 2>&1; echo "rc=$?" >> gpurun_out/t44_all.log
timeout -k 5 300 python scripts/gemm_shapes.py --model D --out gpurun_out/gemm_shapes44_D.json > gpurun_out/gemm_shapes44_D.log 2>&1
timeout -k 10 900 python bench.py --model D --steps 3 --warmup 3 --no-codec --no-cpu-baseline > gpurun_out/b44_D.log 2>&1; echo "rc=$?" >> gpurun_out/b44_D.log
timeout -k 10 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b44_C.log 2>&1; echo "rc=$?" >> gpurun_out/b44_C.log
