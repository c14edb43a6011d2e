#!/bin/bash
# GPU box: the default bench line, then the visit-pair ncu launch list and one --set full capture
# (each only after the same program exited 0 without ncu); outputs under gpurun_out/ (tag $1)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TAG=${1:-r02b}
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; tail -c 400 gpurun_out/${TAG}_bench.json
timeout 300 python scripts/ncu_visit.py > gpurun_out/${TAG}_visit.log 2>&1 && echo "visit ok" || { echo "visit failed"; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/${TAG}_visit_launches.csv python scripts/ncu_visit.py > gpurun_out/${TAG}_ncu1.log 2>&1
echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -o gpurun_out/${TAG}_visit_full -f python scripts/ncu_visit.py > gpurun_out/${TAG}_ncu2.log 2>&1
echo "ncu full rc=$?"
ncu -i gpurun_out/${TAG}_visit_full.ncu-rep --page raw --csv 2>/dev/null | python scripts/ncu_extract.py > gpurun_out/${TAG}_visit_full.csv
rm -f gpurun_out/${TAG}_visit_full.ncu-rep
wc -l gpurun_out/${TAG}_visit_full.csv
