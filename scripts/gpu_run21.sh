# stream-K GEMM tail: numerics, per-shape timing on/off, 1-GPU bench
python -c "import paper_2301_11913_b200._lib as L; print(\"pair_clusters\", L.lib().swarm_gemm_pair_clusters())" > gpurun_out/clusters21.log 2>&1
cd $GRAFT_REPO_ROOT
timeout -k 5 400 python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider > gpurun_out/t21_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/t21_gemm.log
timeout -k 5 210 python scripts/gemm_shapes.py --out gpurun_out/gemm_shapes21_sk.json > gpurun_out/gemm_shapes21_sk.log 2>&1
SWARM_GEMM_STREAMK=0 timeout -k 5 210 python scripts/gemm_shapes.py --out gpurun_out/gemm_shapes21_dp.json > gpurun_out/gemm_shapes21_dp.log 2>&1
timeout -k 5 600 python -m pytest tests/test_stage_gpu.py tests/test_pipeline_gpu.py -x -q -p no:cacheprovider > gpurun_out/t21_stage.log 2>&1; echo "rc=$?" >> gpurun_out/t21_stage.log
timeout -k 10 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b21_C.log 2>&1; echo "rc=$?" >> gpurun_out/b21_C.log
