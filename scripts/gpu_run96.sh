cd $GRAFT_REPO_ROOT
for L in 1 2; do
timeout -k 10 1200 python bench.py --model D --workload engine --lanes $L > gpurun_out/b96_D_n1_l$L.log 2>&1; echo "rc=$?" >> gpurun_out/b96_D_n1_l$L.log
done
