cd $GRAFT_REPO_ROOT
timeout -k 5 300 python scripts/gemm_shapes.py --model C > gpurun_out/gs80_C.log 2>&1
SWARM_GEMM_MCAST=0 timeout -k 5 300 python scripts/gemm_shapes.py --model C > gpurun_out/gs80_C_nomc.log 2>&1
timeout -k 5 300 python scripts/gemm_shapes.py --model D > gpurun_out/gs80_D.log 2>&1
