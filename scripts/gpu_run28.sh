cd $GRAFT_REPO_ROOT
python -c "import paper_2301_11913_b200._lib as L; print('pair', L.lib().swarm_gemm_pair_clusters())" > gpurun_out/clusters28.log 2>&1
SWARM_GEMM_MCAST=1 python -c "import paper_2301_11913_b200._lib as L; print('quad', L.lib().swarm_gemm_pair_clusters())" >> gpurun_out/clusters28.log 2>&1
timeout -k 5 300 python scripts/gemm_shapes.py --out gpurun_out/gemm_shapes28.json > gpurun_out/gemm_shapes28.log 2>&1
SWARM_GEMM_MCAST=1 timeout -k 5 300 python scripts/gemm_shapes.py --out gpurun_out/gemm_shapes28_mc.json > gpurun_out/gemm_shapes28_mc.log 2>&1
