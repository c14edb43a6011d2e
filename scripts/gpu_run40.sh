cd $GRAFT_REPO_ROOT
timeout -k 5 120 python scripts/launch_overhead.py > gpurun_out/launch40.log 2>&1
SWARM_PDL=0 timeout -k 5 120 python scripts/launch_overhead.py >> gpurun_out/launch40.log 2>&1
