#!/bin/bash
# compute-sanitizer over the small all-ops workload (tools/sanitize_ops.py) and smoke():
# memcheck, racecheck, synccheck, initcheck. Summaries -> gpurun_out/${TAG}_sanitize_*.log
TAG=${1:-r2}
O=gpurun_out; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  timeout 1500 $CS --tool $tool $extra --error-exitcode 17 --print-limit 50 \
    python tools/sanitize_ops.py > $O/${TAG}_sanitize_${tool}.log 2>&1
  echo "rc=$?" >> $O/${TAG}_sanitize_${tool}.log
done
timeout 600 $CS --tool memcheck --error-exitcode 17 python -c "import __graft_entry__ as g; g.smoke()" \
  > $O/${TAG}_sanitize_smoke.log 2>&1; echo "rc=$?" >> $O/${TAG}_sanitize_smoke.log
