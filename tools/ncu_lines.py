#!/usr/bin/env python3
"""Per-CUDA-source-line totals (stall samples, instructions) from
`ncu --page source --csv --print-source cuda,sass`.
usage: python tools/ncu_lines.py source.csv [function-substring] [top]"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    sub = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    fname, func, hdr = None, None, None
    cur_line = None
    acc = collections.defaultdict(lambda: [0, 0, "", collections.Counter()])
    total = collections.Counter()
    for row in csv.reader(open(path)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] == "Function Name":
            func = row[1]
            continue
        if row[0] == "Line No":
            hdr = row
            ix = {h: i for i, h in enumerate(hdr) if i >= 2}
            continue
        if hdr is None or sub not in (func or ""):
            continue
        if row[0]:
            cur_line = (fname, int(row[0]), row[1].strip()[:90])
            continue
        if not row[2].startswith("0x"):
            continue
        smp = int(row[4] or 0)
        ins = int(row[7] or 0) if row[7].isdigit() else 0
        a = acc[cur_line]
        a[0] += smp
        a[1] += ins
        for h, i in ix.items():
            if h.startswith("stall_") and "Not Issued" not in h and row[i].isdigit() and int(row[i]):
                a[3][h[6:]] += int(row[i])
        total["s"] += smp
        total["i"] += ins
    print(f"function filter '{sub}': samples={total['s']} instructions={total['i'] / 1e9:.3f} G")
    for k, a in sorted(acc.items(), key=lambda kv: -kv[1][0])[:top]:
        st = " ".join(f"{n}={v}" for n, v in a[3].most_common(3))
        print(f"{100 * a[0] / max(1, total['s']):5.1f}% {100 * a[1] / max(1, total['i']):5.1f}%i {k[0]}:{k[1]} {k[2][:70]} | {st}")


if __name__ == "__main__":
    main()
