cd $GRAFT_REPO_ROOT
timeout -k 5 600 python -m pytest tests/test_norm_gpu.py tests/test_stage_gpu.py -x -q -p no:cacheprovider > gpurun_out/t43.log 2>&1; echo "rc=$?" >> gpurun_out/t43.log
timeout -k 5 120 python scripts/ln_time.py > gpurun_out/ln43.log 2>&1
timeout -k 10 900 python bench.py --model D --steps 3 --warmup 3 --no-codec > gpurun_out/b43_D.log 2>&1; echo "rc=$?" >> gpurun_out/b43_D.log
for mb in 1 2 8; do timeout -k 10 600 python bench.py --micro-batch $mb --steps 3 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b43_C_mb$mb.log 2>&1; echo "rc=$?" >> gpurun_out/b43_C_mb$mb.log; done
timeout -k 10 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b43_C.log 2>&1; echo "rc=$?" >> gpurun_out/b43_C.log
