cd $GRAFT_REPO_ROOT
( time timeout -k 10 900 python bench.py ) > gpurun_out/b36_default.log 2>&1; echo "rc=$?" >> gpurun_out/b36_default.log
( time timeout -k 10 900 python bench.py --impl reference ) > gpurun_out/b36_ref.log 2>&1; echo "rc=$?" >> gpurun_out/b36_ref.log
timeout -k 5 120 python scripts/ln_time.py > gpurun_out/ln36.log 2>&1
SWARM_PDL=0 timeout -k 5 120 python scripts/ln_time.py >> gpurun_out/ln36.log 2>&1
