cd $GRAFT_REPO_ROOT
for m in 0 8 16 32 64 128 443; do echo "mult=$m" >> gpurun_out/deq61.log; SWARM_DEQ_GRID_MULT=$m timeout -k 5 300 python scripts/deq_probe.py 2>&1 | grep k_dequant >> gpurun_out/deq61.log; done
