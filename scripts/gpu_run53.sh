cd $GRAFT_REPO_ROOT
timeout -k 5 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t53_all.log 2>&1; echo "rc=$?" >> gpurun_out/t53_all.log
timeout -k 5 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke53.log 2>&1; echo "rc=$?" >> gpurun_out/smoke53.log
timeout -k 10 900 python bench.py > gpurun_out/b53_n1.log 2>&1; echo "rc=$?" >> gpurun_out/b53_n1.log
