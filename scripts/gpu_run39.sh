# round-1 profiles of the default bench path: launch list (shares) and one full ncu capture of k_gemm2
cd $GRAFT_REPO_ROOT
timeout -k 10 600 python bench.py --steps 2 --warmup 3 --microbatches 8 --no-cpu-baseline --no-codec > gpurun_out/b39_pre.log 2>&1; echo "rc=$?" >> gpurun_out/b39_pre.log
timeout -k 10 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches39.csv python bench.py --steps 2 --warmup 3 --microbatches 8 --no-cpu-baseline --no-codec > gpurun_out/ncu39_launch.log 2>&1; echo "rc=$?" >> gpurun_out/ncu39_launch.log
timeout -k 10 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm2 --launch-skip 60 --launch-count 4 -o gpurun_out/ncu_gemm39 python bench.py --steps 1 --warmup 3 --microbatches 8 --no-cpu-baseline --no-codec > gpurun_out/ncu39_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/ncu39_gemm.log
