#!/usr/bin/env python3
"""profiles/ncu_traffic.json from an `ncu --set full` raw export of the bench's
hot kernels: per launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum)
and executed warp instructions (smsp__inst_executed.sum), keyed by the bench's
profiling names. usage: python tools/ncu_traffic.py RAW_CSV ABOUT > profiles/ncu_traffic.json"""
import csv
import json
import sys

# kernel name -> the bench's profiling scope (first match wins)
NAMES = [("select_stream_kernel<2, 1>", "sum_stream"), ("select_stream_kernel<", "select_stream"),
         ("project_stream_kernel", "project_stream"), ("pos_copy_kernel<32>", "project_copy"),
         ("pos_copy_kernel<8>", "pos_copy"), ("pos_slot_kernel<2>", "pos_slot+"), ("pos_slot_kernel", "pos_slot")]


def scale(v, unit):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return float(v.replace(",", "")) * f


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if r]
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    acc = {}
    for r in rows[2:]:
        name = r[ix["Kernel Name"]]
        key = next((k for s, k in NAMES if s in name), None)
        if key is None:
            continue
        rd = scale(r[ix["dram__bytes_read.sum"]], units[ix["dram__bytes_read.sum"]])
        wr = scale(r[ix["dram__bytes_write.sum"]], units[ix["dram__bytes_write.sum"]])
        ins = float(r[ix["smsp__inst_executed.sum"]].replace(",", ""))
        a = acc.setdefault(key, [0.0, 0.0, 0])
        a[0] += rd + wr
        a[1] += ins
        a[2] += 1
    # pos_slot: the dense launch plus the deferred-blocks launch form one encoder step
    extra = acc.pop("pos_slot+", None)
    out = {"_about": sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]}
    inst = {}
    for k, (b, ins, c) in acc.items():
        if k == "pos_slot" and extra:
            b, ins = b + extra[0], ins + extra[1]
        out[k] = int(b / c)
        inst[k] = int(ins / c)
    out["_inst"] = inst
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
