cd $GRAFT_REPO_ROOT
timeout -k 5 600 python -m pytest tests/test_codec_gpu.py tests/test_compat_gpu.py -x -q -p no:cacheprovider > gpurun_out/t59_codec.log 2>&1; echo "rc=$?" >> gpurun_out/t59_codec.log
timeout -k 5 300 python scripts/deq_probe.py > gpurun_out/deq59.log 2>&1; echo "rc=$?" >> gpurun_out/deq59.log
timeout -k 5 600 ncu --set full --clock-control none --import-source on -k regex:k_dequant_blocks -c 1 -o gpurun_out/ncu_deq59 python scripts/deq_probe.py > gpurun_out/ncu_deq59.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_deq59.log
timeout -k 10 600 python bench.py --workload codec > gpurun_out/b59_codec.log 2>&1; echo "rc=$?" >> gpurun_out/b59_codec.log
