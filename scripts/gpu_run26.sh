cd $GRAFT_REPO_ROOT
timeout -k 5 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t26_all.log 2>&1; echo "rc=$?" >> gpurun_out/t26_all.log
timeout -k 10 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b26_C.log 2>&1; echo "rc=$?" >> gpurun_out/b26_C.log
SWARM_PDL=0 timeout -k 10 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b26_C_nopdl.log 2>&1; echo "rc=$?" >> gpurun_out/b26_C_nopdl.log
timeout -k 5 210 python scripts/gemm_shapes.py --out gpurun_out/gemm_shapes26.json > gpurun_out/gemm_shapes26.log 2>&1
