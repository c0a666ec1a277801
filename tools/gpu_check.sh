#!/bin/bash
# One GPU-box pass: gpu tests, smoke, default bench, launch list, ncu full of the top kernels.
# usage (from the repo root, under gpurun): [NCU=regex] bash tools/gpu_check.sh TAG
TAG=${1:-run}
O=gpurun_out
mkdir -p $O
if [ -z "$NO_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -x -q > $O/${TAG}_gpu_tests.log 2>&1; echo rc=$? >> $O/${TAG}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo rc=$? >> $O/${TAG}_smoke.log
fi
timeout 900 python bench.py $BENCH_ARGS > $O/${TAG}_bench.log 2>&1; echo rc=$? >> $O/${TAG}_bench.log
if [ -n "$NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu $BENCH_ARGS > $O/${TAG}_ncu_l.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$NCU" -s ${NCU_SKIP:-6} -c ${NCU_COUNT:-3} \
  -o /tmp/${TAG}_prof python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu $BENCH_ARGS > $O/${TAG}_ncu_full.log 2>&1
ncu -i /tmp/${TAG}_prof.ncu-rep --page raw --csv > $O/${TAG}_raw.csv 2>&1
ncu -i /tmp/${TAG}_prof.ncu-rep --page details --csv > $O/${TAG}_details.csv 2>&1
if [ -n "$NCU_SOURCE" ]; then
ncu -i /tmp/${TAG}_prof.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${TAG}_source.csv 2>&1
python tools/ncu_lines.py /tmp/${TAG}_source.csv "" 60 > $O/${TAG}_lines.txt 2>&1
fi
sz=$(stat -c %s /tmp/${TAG}_prof.ncu-rep)
if [ "$sz" -lt 20000000 ]; then cp /tmp/${TAG}_prof.ncu-rep $O/; fi
fi
du -sh $O
echo done
