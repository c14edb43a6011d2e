cd $GRAFT_REPO_ROOT
for d in 0 8; do SWARM_GEMM_DBG=$d timeout -k 5 120 python scripts/streamk_diag.py >> gpurun_out/skdiag23.log 2>&1; done
timeout -k 5 300 python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider > gpurun_out/t23_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/t23_gemm.log
