# ncu launch list (gpu__time_duration per launch) of a command; usage: bash tools/ncu_launches.sh TAG cmd...
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv "$@" > gpurun_out/${TAG}_ncu_l.log 2>&1
python - gpurun_out/${TAG}_launches.csv <<'PY' > gpurun_out/${TAG}_launches.txt
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
acc = collections.defaultdict(list)
for r in rows[1:]:
    try: acc[r[ki][:90]].append(float(r[vi].replace(",", "")))
    except ValueError: pass
for k, v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
    print(f"{len(v):4d} {sum(v)/len(v)/1000:9.3f} us avg  {k}")
PY
