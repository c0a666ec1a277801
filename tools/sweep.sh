#!/bin/bash
# env-variant sweep of the default bench (kernel times only): bash tools/sweep.sh TAG "ENV1" "ENV2" ...
TAG=$1; shift
O=gpurun_out; mkdir -p $O
for V in "$@"; do
  echo "=== $V" >> $O/${TAG}_sweep.log
  env $V timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu $BENCH_ARGS 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('step_ms', round(d['ms_per_step'],3), ' '.join(f\"{k}={v['avg_ms']:.3f}\" for k,v in d['kernels'].items()))" >> $O/${TAG}_sweep.log 2>&1
done
echo done >> $O/${TAG}_sweep.log
