cd $GRAFT_REPO_ROOT
timeout -k 5 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t62_all.log 2>&1; echo "rc=$?" >> gpurun_out/t62_all.log
timeout -k 10 1200 python bench.py > gpurun_out/b62_n1.log 2>&1; echo "rc=$?" >> gpurun_out/b62_n1.log
timeout -k 10 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches62.csv python bench.py --steps 2 --warmup 3 --microbatches 8 --no-codec --no-engine --no-cpu-baseline > gpurun_out/ncu62.log 2>&1; echo "rc=$?" >> gpurun_out/ncu62.log
