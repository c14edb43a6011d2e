cd $GRAFT_REPO_ROOT
timeout -k 5 600 python -m pytest tests/test_executor_gpu.py -x -q -p no:cacheprovider > gpurun_out/t55_exec.log 2>&1; echo "rc=$?" >> gpurun_out/t55_exec.log
timeout -k 10 900 python bench.py --workload engine --no-cpu-baseline > gpurun_out/b55_engine_n1.log 2>&1; echo "rc=$?" >> gpurun_out/b55_engine_n1.log
