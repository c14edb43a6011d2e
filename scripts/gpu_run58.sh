cd $GRAFT_REPO_ROOT
timeout -k 5 300 python scripts/deq_probe.py > gpurun_out/deq58.log 2>&1; echo "rc=$?" >> gpurun_out/deq58.log
timeout -k 5 600 ncu --set full --clock-control none --import-source on -k regex:k_dequant_words -c 1 -o gpurun_out/ncu_deq58 python scripts/deq_probe.py > gpurun_out/ncu_deq58.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_deq58.log
