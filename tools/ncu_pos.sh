# ncu --set full of one pos_slot launch (select X<2^16 -> DELTA_BP{512} at 2^30 rows, c5-shaped X),
# per-source-line totals. usage (under gpurun): bash tools/ncu_pos.sh TAG [kernel-regex]
TAG=${1:-pos}; K=${2:-pos_slot}; LG=${3:-30}
O=gpurun_out; mkdir -p $O
REPS=3 timeout 300 python tools/prof_sel.py $LG > $O/${TAG}_prof.log 2>&1
timeout 600 ncu -f --set full --clock-control none --import-source on --kernel-name-base ${KBASE:-function} -k regex:$K -s 1 -c 1 -o /tmp/${TAG} python tools/prof_sel.py $LG > $O/${TAG}_ncu.log 2>&1
ncu -i /tmp/${TAG}.ncu-rep --page raw --csv > $O/${TAG}_raw.csv 2>&1
ncu -i /tmp/${TAG}.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${TAG}_source.csv 2>&1
python tools/ncu_lines.py /tmp/${TAG}_source.csv "" 50 > $O/${TAG}_lines.txt 2>&1
