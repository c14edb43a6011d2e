# driver-like checks: full GPU suite, smoke, default bench (cpu baseline + codec), reference arm, codec workload
cd $GRAFT_REPO_ROOT
timeout -k 5 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t35_all.log 2>&1; echo "rc=$?" >> gpurun_out/t35_all.log
timeout -k 5 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke35.log 2>&1; echo "rc=$?" >> gpurun_out/smoke35.log
/usr/bin/time -v timeout -k 10 900 python bench.py > gpurun_out/b35_default.log 2> gpurun_out/b35_default.err; echo "rc=$?" >> gpurun_out/b35_default.log
timeout -k 10 900 python bench.py --impl reference > gpurun_out/b35_ref.log 2>&1; echo "rc=$?" >> gpurun_out/b35_ref.log
timeout -k 10 600 python bench.py --workload codec > gpurun_out/b35_codec.log 2>&1; echo "rc=$?" >> gpurun_out/b35_codec.log
