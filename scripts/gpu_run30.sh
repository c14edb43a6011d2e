cd $GRAFT_REPO_ROOT
timeout -k 5 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t30_all.log 2>&1; echo "rc=$?" >> gpurun_out/t30_all.log
timeout -k 5 120 python scripts/ln_time.py > gpurun_out/ln30.log 2>&1
