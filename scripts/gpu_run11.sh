cd $GRAFT_REPO_ROOT
timeout -k 5 120 python -m pytest tests/test_attention_gpu.py -q -x -p no:cacheprovider > gpurun_out/t11_attn.log 2>&1; echo "rc=$?" >> gpurun_out/t11_attn.log
timeout -k 5 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t11_all.log 2>&1; echo "rc=$?" >> gpurun_out/t11_all.log
timeout -k 10 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b11_C.log 2>&1; echo "rc=$?" >> gpurun_out/b11_C.log
SWARM_ATTN_FUSED=0 timeout -k 10 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b11_C_unfused.log 2>&1; echo "rc=$?" >> gpurun_out/b11_C_unfused.log
