cd $GRAFT_REPO_ROOT
timeout -k 10 400 python scripts/host_overhead.py C > gpurun_out/host6.log 2>&1; echo "rc=$?" >> gpurun_out/host6.log
