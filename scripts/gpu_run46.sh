cd $GRAFT_REPO_ROOT
timeout -k 5 120 python scripts/streamk_diag_D.py > gpurun_out/skD46.log 2>&1
SWARM_GEMM_STREAMK=1 timeout -k 5 120 python scripts/streamk_diag_D.py >> gpurun_out/skD46.log 2>&1
SWARM_GEMM_DBG=8 timeout -k 5 120 python scripts/streamk_diag_D.py >> gpurun_out/skD46.log 2>&1
