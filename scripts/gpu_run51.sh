cd $GRAFT_REPO_ROOT
timeout -k 5 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t51_all.log 2>&1; echo "rc=$?" >> gpurun_out/t51_all.log
timeout -k 10 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b51_C.log 2>&1; echo "rc=$?" >> gpurun_out/b51_C.log
timeout -k 10 900 python bench.py --model D --steps 3 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b51_D.log 2>&1; echo "rc=$?" >> gpurun_out/b51_D.log
