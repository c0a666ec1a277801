# ncu --set full of one kernel launch of a prof_ops target, with the per-line summary
# usage: bash tools/run_ncu_one.sh TAG KERNEL_REGEX SKIP TARGET
TAG=$1; K=$2; S=$3; T=$4
O=gpurun_out; mkdir -p $O
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:$K -s $S -c ${COUNT:-1} -o /tmp/$TAG python tools/prof_ops.py $T > $O/${TAG}_ncu.log 2>&1
ncu -i /tmp/$TAG.ncu-rep --page raw --csv > $O/${TAG}_raw.csv 2>&1
ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src.csv 2>&1
python tools/ncu_lines.py /tmp/src.csv "" 50 > $O/${TAG}_lines.txt 2>&1
