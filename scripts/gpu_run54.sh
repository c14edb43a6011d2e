cd $GRAFT_REPO_ROOT
timeout -k 5 600 python -m pytest tests/test_codec_gpu.py tests/test_compat_gpu.py -x -q -p no:cacheprovider > gpurun_out/t54_codec.log 2>&1; echo "rc=$?" >> gpurun_out/t54_codec.log
timeout -k 10 600 python bench.py --workload codec > gpurun_out/b54_codec.log 2>&1; echo "rc=$?" >> gpurun_out/b54_codec.log
