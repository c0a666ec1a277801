#!/usr/bin/env python3
"""Top stalled SASS instructions per kernel from `ncu --page source --csv --print-source sass`.
usage: python tools/ncu_hot.py source.csv [kernel-substring] [top]"""
import csv
import io
import sys


def sections(path):
    cur = None
    for line in open(path):
        if line.startswith('"Kernel Name"'):
            if cur:
                yield cur
            cur = [line.split('","', 1)[1].rstrip(',\n').strip('"'), []]
        elif cur is not None:
            cur[1].append(line)
    if cur:
        yield cur


def main():
    path = sys.argv[1]
    sub = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    seen = set()
    for name, body in sections(path):
        if sub not in name or name in seen:
            continue
        seen.add(name)
        rows = list(csv.reader(io.StringIO("".join(body))))
        hdr = rows[0]
        ix = {h: i for i, h in enumerate(hdr)}
        data = [r for r in rows[1:] if len(r) == len(hdr)]
        S = ix["Warp Stall Sampling (All Samples)"]
        tot = sum(int(r[S] or 0) for r in data) or 1
        print(f"== {name[:150]}\n   samples={tot} instrs={len(data)}")
        stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        for r in sorted(data, key=lambda r: -int(r[S] or 0))[:top]:
            s = int(r[S] or 0)
            st = " ".join(f"{c[6:]}={r[ix[c]]}" for c in stall_cols if r[ix[c]] not in ("0", ""))
            print(f"{r[0][-5:]} {100 * s / tot:5.1f}% {r[1].strip()[:58]:58s} ex={r[ix['Instructions Executed']]} "
                  f"conf={r[ix['L1 Conflicts Shared N-Way']]} {st}")


if __name__ == "__main__":
    main()
