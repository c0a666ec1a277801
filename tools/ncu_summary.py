#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and an
`ncu --set full` details page (--page details --csv) into markdown.
usage: python tools/ncu_summary.py TAG [gpurun_out] > profiles/TAG.md"""
import collections
import csv
import os
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "L2 Hit Rate", "Achieved Occupancy", "Registers Per Thread", "Grid Size",
        "Block Size", "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction"]


def rows_after_header(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    return rows[i], rows[i + 1:]


def main():
    tag = sys.argv[1]
    d = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
    print(f"# ncu summary `{tag}`\n")
    lp = os.path.join(d, f"{tag}_launches.csv")
    if os.path.exists(lp):
        hdr, rows = rows_after_header(lp)
        agg = collections.defaultdict(lambda: [0, 0.0])
        # launches before the first select are the bench's setup (input generation and
        # compression of X and Y, outside the timed region): listed apart
        started = not any(any(s in dict(zip(hdr, r)).get("Kernel Name", "") for s in ("select_fast", "select_stream")) for r in rows)
        for r in rows:
            x = dict(zip(hdr, r))
            if x.get("Metric Name") == "gpu__time_duration.sum":
                unit = x["Metric Unit"]
                v = float(x["Metric Value"].replace(",", ""))
                v = v / 1e3 if unit == "ns" else v * 1e3 if unit == "ms" else v  # -> us
                started = started or "select_fast" in x["Kernel Name"] or "select_stream" in x["Kernel Name"]
                k = x["Kernel Name"].split("(")[0][:90] + ("" if started else " [setup]")
                agg[k][0] += 1
                agg[k][1] += v
        ours_k = lambda k: (k.startswith("void ms::") or k.startswith("ms::")) and not k.endswith("[setup]")
        tot = sum(v[1] for k, v in agg.items() if ours_k(k))
        print("## Launch list (`--metrics gpu__time_duration.sum --clock-control none`, cold, serialised)\n")
        print("| kernel | launches | total us | avg us | share of libms time |\n|---|---|---|---|---|")
        for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            ours = ours_k(k)
            share = f"{100 * t / tot:.1f}%" if ours and tot else "(setup / torch)"
            print(f"| `{k}` | {c} | {t:.1f} | {t / c:.1f} | {share} |")
        print()
    dp = os.path.join(d, f"{tag}_details.csv")
    if os.path.exists(dp):
        hdr, rows = rows_after_header(dp)
        per = collections.OrderedDict()
        for r in rows:
            x = dict(zip(hdr, r))
            key = (x["ID"], x["Kernel Name"].split("(")[0][:90])
            if x.get("Metric Name") in KEYS:
                per.setdefault(key, {})[x["Metric Name"]] = f'{x["Metric Value"]} {x["Metric Unit"]}'.strip()
        print("## `ncu --set full` captures\n")
        print("| id | kernel | " + " | ".join(KEYS) + " |")
        print("|" + "---|" * (len(KEYS) + 2))
        for (i, k), m in per.items():
            print(f"| {i} | `{k}` | " + " | ".join(m.get(q, "") for q in KEYS) + " |")
        print()
    rp = os.path.join(d, f"{tag}_raw.csv")
    if os.path.exists(rp):
        rows = list(csv.reader(open(rp)))
        hdr = rows[0]
        ix = {h: i for i, h in enumerate(hdr)}
        want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"]
        if all(w in ix for w in want):
            print("## DRAM traffic per captured launch (`--set full`, raw page)\n")
            print("| id | kernel | dram read | dram write | duration |\n|---|---|---|---|---|")
            units = rows[1]
            for r in rows[2:]:
                if len(r) < len(hdr):
                    continue
                print(f"| {r[ix['ID']]} | `{r[ix['Kernel Name']].split('(')[0][:80]}` | "
                      + " | ".join(f"{r[ix[w]]} {units[ix[w]]}" for w in want) + " |")
            print()


if __name__ == "__main__":
    main()
