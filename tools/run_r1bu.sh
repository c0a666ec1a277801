O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q -k "morph or compress or static" > $O/r1bu_tests.log 2>&1; echo rc=$? >> $O/r1bu_tests.log
timeout 300 python tools/prof_ops.py c3 > $O/r1bu_prof.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:engine_kernel -c 5 -o /tmp/eng python tools/prof_ops.py c3e > $O/r1bu_ncu.log 2>&1
ncu -i /tmp/eng.ncu-rep --page raw --csv > $O/r1bu_raw.csv 2>&1
ncu -i /tmp/eng.ncu-rep --page details --csv > $O/r1bu_details.csv 2>&1
ncu -i /tmp/eng.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src.csv 2>&1
python tools/ncu_lines.py /tmp/src.csv "" 60 > $O/r1bu_lines.txt 2>&1
du -sh $O
