cd $GRAFT_REPO_ROOT
timeout -k 5 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t41_all.log 2>&1; echo "rc=$?" >> gpurun_out/t41_all.log
timeout -k 5 120 python scripts/ln_time.py > gpurun_out/ln41.log 2>&1
timeout -k 10 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b41_C.log 2>&1; echo "rc=$?" >> gpurun_out/b41_C.log
