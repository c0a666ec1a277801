#!/usr/bin/env python3
"""The paper's single-operator experiment (Figure `fig:select`)
on B200: select of the column's lowest value (point predicate, 90% selectivity,
P:569-570) on the synthetic columns C1-C4 (Table `tab:datach`; recipes
in synth/) for all 25 combinations of input and output
format among the five the paper uses (uncompressed, static BP, SIMD-BP512 =
DYN_BP{512}, FOR + BP512, DELTA + BP512).

Every combination is first checked byte-exact against the oracle on the first
2^18 rows, then timed at the paper's 2^27 rows (CUDA events around ms_select,
median of --reps, L2 flushed). Prints one JSON line per combination and a
summary per column: the fastest pair, and its speed-up over uncompressed ->
uncompressed (the paper reports 72-81% runtime savings on its CPU).

usage: python tools/select_sweep.py [--log2n 27] [--reps 5]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import synth  # noqa: E402
from paper_2004_09350_b200 import ms  # noqa: E402

FORMATS = [("UNCOMPR", lambda: ms.uncompr(), (O.UNCOMPR, 0, 0)),
           ("STATIC_BP", lambda: ms.static_bp(0), (O.STATIC_BP, 0, 0)),
           ("DYN_BP512", lambda: ms.dyn_bp(512), (O.DYN_BP, 0, 512)),
           ("FOR_BP512", lambda: ms.for_bp(512), (O.FOR_BP, 0, 512)),
           ("DELTA_BP512", lambda: ms.delta_bp(512), (O.DELTA_BP, 0, 512))]
COLUMNS = ["C1.X", "C2.X", "C3.X", "C4.X"]  # C4: the sorted column


def column(name, n):
    v = synth.gen_host(name, n)
    return v, int(v.min())


def to_dev(v):
    return torch.from_numpy(np.ascontiguousarray(v).view(np.int64)).cuda()


def parity(name, n=1 << 18):
    v, lo = column(name, n)
    t = to_dev(v)
    for fin, mk_in, oin in FORMATS:
        gi = ms.compress(t, mk_in())
        oi = O.encode(v, *oin)
        for fout, mk_out, oout in FORMATS:
            g = ms.select(gi, ms.EQ, lo, out_fmt=mk_out())
            o = O.select(oi, O.EQ, lo, out_fmt=oout[0], out_width=0, out_block=oout[2] or 512)
            img = g.images()
            for sec in ("payload", "cw", "ref", "rem"):
                if not np.array_equal(img[sec], getattr(o, sec)):
                    raise SystemExit(f"parity failure: {name} {fin} -> {fout} section {sec}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2n", type=int, default=27)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    n = 1 << a.log2n
    summary = {}
    for name in COLUMNS:
        parity(name)
        v, lo = column(name, n)
        t = to_dev(v)
        del v
        res = {}
        for fin, mk_in, _ in FORMATS:
            gi = ms.compress(t, mk_in())
            for fout, mk_out, _ in FORMATS:
                ms.select(gi, ms.EQ, lo, out_fmt=mk_out())
                ts = []
                out_bytes = 0
                for _ in range(a.reps):
                    flush.fill_(1)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    e0.record()
                    g = ms.select(gi, ms.EQ, lo, out_fmt=mk_out())
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
                    out_bytes = g.footprint()
                    sel = g.n
                    del g
                t_ms = statistics.median(ts)
                res[(fin, fout)] = t_ms
                print(json.dumps({"column": name, "in": fin, "out": fout, "ms": round(t_ms, 4), "n": n,
                                  "selected": sel, "in_bytes": gi.footprint(), "out_bytes": out_bytes,
                                  "Grows_per_s": round(n / (t_ms * 1e-3) / 1e9, 1)}), flush=True)
            del gi
            torch.cuda.empty_cache()
        base = res[("UNCOMPR", "UNCOMPR")]
        best = min(res, key=res.get)
        summary[name] = {"uncompr_ms": round(base, 4), "best": list(best), "best_ms": round(res[best], 4),
                         "saving_pct": round(100 * (1 - res[best] / base), 1),
                         "worst": list(max(res, key=res.get)), "worst_ms": round(max(res.values()), 4)}
        del t
        torch.cuda.empty_cache()
    print(json.dumps({"summary": summary}), flush=True)


if __name__ == "__main__":
    main()
