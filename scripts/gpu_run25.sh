cd $GRAFT_REPO_ROOT
timeout -k 10 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b25_C.log 2>&1; echo "rc=$?" >> gpurun_out/b25_C.log
timeout -k 10 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 3000 --csv --log-file gpurun_out/launches25_warm.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-codec --microbatches 8 > gpurun_out/ncu25.log 2>&1; echo "rc=$?" >> gpurun_out/ncu25.log
