cd $GRAFT_REPO_ROOT
timeout -k 5 200 python scripts/wgrad_pair_probe.py > gpurun_out/wgrad50.log 2>&1
