#!/usr/bin/env python3
"""Print selected metrics of an `ncu --page raw --csv` export, one block per launch.
usage: python tools/rawpick.py raw.csv [metric-substring ...]"""
import csv
import sys

DEFAULT = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "dram__bytes_read.sum",
           "dram__bytes_write.sum", "Kernel Name"]
rows = [r for r in csv.reader(open(sys.argv[1])) if r]
h = rows[0]
want = sys.argv[2:] or DEFAULT
for r in rows[2:]:
    for i, x in enumerate(h):
        if any(w == x for w in want) or (sys.argv[2:] and any(w in x for w in want)):
            print(f"{x} = {r[i]}")
    print("--")
