cd $GRAFT_REPO_ROOT
timeout -k 5 120 python scripts/attn_trace.py > gpurun_out/attn_trace33.log 2>&1
