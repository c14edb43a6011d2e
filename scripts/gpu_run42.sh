cd $GRAFT_REPO_ROOT
timeout -k 5 600 python -m pytest tests/test_norm_gpu.py tests/test_stage_gpu.py -x -q -p no:cacheprovider > gpurun_out/t42.log 2>&1; echo "rc=$?" >> gpurun_out/t42.log
timeout -k 5 120 python scripts/ln_time.py > gpurun_out/ln42.log 2>&1
timeout -k 5 300 ncu --set full --import-source on --clock-control none -k regex:k_ln -c 3 -o gpurun_out/ncu_ln42 python scripts/ln_time.py > gpurun_out/ncu_ln42.log 2>&1
