cd $GRAFT_REPO_ROOT
timeout -k 5 300 python scripts/gemm_shapes.py --model D > gpurun_out/gs81_D.log 2>&1
SWARM_GEMM_SMALL=60 timeout -k 5 300 python scripts/gemm_shapes.py --model D > gpurun_out/gs81_D_small60.log 2>&1
SWARM_GEMM_SMALL=100 timeout -k 5 300 python scripts/gemm_shapes.py --model C > gpurun_out/gs81_C_small100.log 2>&1
