cd $GRAFT_REPO_ROOT
B="python bench.py --steps 1 --warmup 3 --microbatches 4 --no-cpu-baseline --no-codec"
timeout -k 10 600 $B > gpurun_out/b10_plain.log 2>&1 && \
timeout -k 10 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 9000 -c 6000 --csv --log-file gpurun_out/launches10.csv $B > gpurun_out/ncu_launch10.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_launch10.log
timeout -k 10 120 python scripts/ncu_gemm_shapes.py && \
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 2 -c 2 -o gpurun_out/ncu_gemm10 python scripts/ncu_gemm_shapes.py > gpurun_out/ncu_gemm10.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_gemm10.log
C="python bench.py --workload codec --steps 30 --warmup 3 --no-cpu-baseline"
timeout -k 10 300 $C > gpurun_out/b10_codec.log 2>&1 && \
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:"k_quant_f32|k_dequant_table" -s 10 -c 2 -o gpurun_out/ncu_codec10 $C > gpurun_out/ncu_codec10.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_codec10.log
