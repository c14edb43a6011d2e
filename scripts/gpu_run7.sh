cd $GRAFT_REPO_ROOT
timeout -k 10 400 python scripts/host_overhead.py C > gpurun_out/host7.log 2>&1; echo "rc=$?" >> gpurun_out/host7.log
timeout -k 10 600 python -m pytest tests/test_pipeline_gpu.py tests/test_stage_gpu.py -q -p no:cacheprovider > gpurun_out/t7.log 2>&1; echo "rc=$?" >> gpurun_out/t7.log
timeout -k 10 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b7_C.log 2>&1; echo "rc=$?" >> gpurun_out/b7_C.log
