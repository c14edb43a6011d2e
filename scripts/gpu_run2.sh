cd $GRAFT_REPO_ROOT
timeout -k 10 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t2_all.log 2>&1; echo "rc=$?" >> gpurun_out/t2_all.log
timeout -k 10 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/b2_plain.log 2>&1 && \
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:k_quant_f32 -s 5 -c 1 -o gpurun_out/ncu_quant python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_quant.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_quant.log
