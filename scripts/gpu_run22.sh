cd $GRAFT_REPO_ROOT
for d in 0 8 16; do SWARM_GEMM_DBG=$d timeout -k 5 120 python scripts/streamk_diag.py >> gpurun_out/skdiag22.log 2>&1; done
timeout -k 5 210 python scripts/gemm_shapes.py --out gpurun_out/gemm_shapes22.json > gpurun_out/gemm_shapes22.log 2>&1
