# codec kernel v2 check: parity tests + bench + ncu of both codec kernels
cd $GRAFT_REPO_ROOT
timeout -k 10 600 python -m pytest tests/test_codec_gpu.py tests/test_stage_gpu.py -q -p no:cacheprovider -x > gpurun_out/t3.log 2>&1; echo "rc=$?" >> gpurun_out/t3.log
timeout -k 10 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/b3_plain.log 2>&1 && \
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:"k_quant_f32|k_dequant_table" -s 10 -c 2 -o gpurun_out/ncu_codec3 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_codec3.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_codec3.log
