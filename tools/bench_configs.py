#!/usr/bin/env python3
"""Per-operator timings of BASELINE.json configs c1..c4 at their full sizes on
one GPU (c5 is bench.py's workload). Every op goes through the C ABI; times are
CUDA events on the current stream around each call (median of --reps after one
warm-up, inputs resident, L2 flushed before each rep by writing 256 MB). Prints
one JSON object per line: config, op, ms, rows/s, and the op's algorithmic bytes
(compressed inputs read + outputs written) as GB/s against MEASURED_PEAKS.json.

usage: python tools/bench_configs.py [--reps 5] [--configs c1,c2,c3,c4]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2004_09350_b200 import ms  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
_flush = None


def flush_l2():
    global _flush
    if _flush is None:
        _flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    _flush.fill_(1)


def timed(fn, reps):
    fn()  # warm-up
    ts = []
    for _ in range(reps):
        flush_l2()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        del out
    return statistics.median(ts)


def report(cfg, op, ms_, rows, alg_bytes):
    line = {"config": cfg, "op": op, "ms": round(ms_, 4), "Grows_per_s": round(rows / (ms_ * 1e-3) / 1e9, 2),
            "alg_bytes": int(alg_bytes), "alg_GBps": round(alg_bytes / (ms_ * 1e-3) / 1e9, 1),
            "frac_of_peak": round(alg_bytes / (ms_ * 1e-3) / 1e9 / PEAK, 3)}
    print(json.dumps(line), flush=True)


def c1(reps):
    n = 1 << 20
    X = ms.compress(synth.gen_torch("c1.X", n), ms.static_bp(10))
    pos = ms.select(X, ms.LT, 102, out_fmt=ms.delta_bp(512))
    report("c1", "select X<102 -> DELTA_BP{512}", timed(lambda: ms.select(X, ms.LT, 102, out_fmt=ms.delta_bp(512)),
                                                       reps), n, X.footprint() + pos.footprint())
    report("c1", "sum X[pos] (fused)", timed(lambda: ms.agg_sum(X, pos), reps), pos.n, X.footprint() + pos.footprint())


def c2(reps):
    n = 1 << 28
    X = ms.compress(synth.gen_torch("c2.X", n), ms.dyn_bp(512))
    Y = ms.compress(synth.gen_torch("c2.Y", n), ms.for_bp(512))
    xu = synth.gen_torch("c2.X", n)
    report("c2", "compress u64 -> DYN_BP{512}", timed(lambda: ms.compress(xu, ms.dyn_bp(512)), reps), n,
           8 * n + X.footprint())
    del xu
    report("c2", "sum X (whole column)", timed(lambda: ms.agg_sum(X), reps), n, X.footprint())
    pos = ms.select(X, ms.EQ, 17, out_fmt=ms.delta_bp(512))
    report("c2", "select X==17 -> DELTA_BP{512}", timed(lambda: ms.select(X, ms.EQ, 17, out_fmt=ms.delta_bp(512)),
                                                        reps), n, X.footprint() + pos.footprint())
    for f, name in ((ms.for_bp(512), "FOR_BP{512}"), (ms.uncompr(), "UNCOMPR")):
        yp = ms.project(Y, pos, 0, f)
        report("c2", f"project Y -> {name}", timed(lambda: ms.project(Y, pos, 0, f), reps), pos.n,
               pos.footprint() + 64 * pos.n + yp.footprint())


def c3(reps):
    n = 1 << 29
    x = synth.gen_torch("c3.x", n)
    R = ms.compress(x, ms.rle())
    D = ms.compress(x, ms.delta_bp(2048))
    del x
    for C, name in ((R, "RLE"), (D, "DELTA_BP{2048}")):
        pos = ms.select(C, ms.BETWEEN, 10**6, 2 * 10**6, out_fmt=ms.delta_bp(512))
        report("c3", f"select {name} in [1e6,2e6) -> DELTA_BP{{512}}",
               timed(lambda: ms.select(C, ms.BETWEEN, 10**6, 2 * 10**6, out_fmt=ms.delta_bp(512)), reps), n,
               C.footprint() + pos.footprint())
        report("c3", f"sum {name} at positions", timed(lambda: ms.agg_sum(C, pos), reps), pos.n,
               pos.footprint() + C.footprint())
    report("c3", "decompress DELTA_BP{2048} -> u64", timed(lambda: ms.decompress(D), reps), n,
           D.footprint() + 8 * n)
    report("c3", "decompress RLE -> u64", timed(lambda: ms.decompress(R), reps), n, R.footprint() + 8 * n)
    xr = ms.decompress(D)
    report("c3", "compress u64 -> DELTA_BP{2048}", timed(lambda: ms.compress(xr, ms.delta_bp(2048)), reps), n,
           8 * n + D.footprint())
    report("c3", "compress u64 -> RLE", timed(lambda: ms.compress(xr, ms.rle()), reps), n, 8 * n + R.footprint())
    del xr
    m1 = ms.morph(R, ms.delta_bp(2048))
    report("c3", "morph RLE -> DELTA_BP{2048}", timed(lambda: ms.morph(R, ms.delta_bp(2048)), reps), n,
           R.footprint() + m1.footprint())
    m2 = ms.morph(D, ms.static_bp(0))
    report("c3", "morph DELTA_BP{2048} -> STATIC_BP{auto}", timed(lambda: ms.morph(D, ms.static_bp(0)), reps), n,
           D.footprint() + m2.footprint())


def c4(reps):
    n = 600_000_000
    Dm = synth.D4
    bm = torch.from_numpy(synth.bitmap_c4().view("int64")).cuda()
    gattr = ms.compress(synth.gen_torch("c4.gattr", Dm[3]), ms.static_bp(10))
    k0 = ms.compress(synth.gen_torch("c4.k0", n), ms.static_bp(12))
    k1 = ms.compress(synth.gen_torch("c4.k1", n), ms.static_bp(18))
    k3 = ms.compress(synth.gen_torch("c4.k3", n), ms.static_bp(17))
    m1 = ms.compress(synth.gen_torch("c4.m1", n), ms.dyn_bp(512))
    m2 = ms.compress(synth.gen_torch("c4.m2", n), ms.dyn_bp(512))

    def chain():
        pos1 = ms.select(k0, ms.BETWEEN, 0, 365, out_fmt=ms.delta_bp(512))
        k1p = ms.project(k1, pos1, 0, ms.static_bp(18))
        idx = ms.select(k1p, ms.IN_BITMAP, bitmap=bm, bitmap_bits=Dm[1], out_fmt=ms.delta_bp(512))
        pos2 = ms.project(pos1, idx, 0, ms.delta_bp(512))
        m1p = ms.project(m1, pos2, 0, ms.dyn_bp(512))
        m2p = ms.project(m2, pos2, 0, ms.dyn_bp(512))
        k3p = ms.project(k3, pos2, 0, ms.static_bp(17))
        gid = ms.project(gattr, k3p, 0, ms.static_bp(10))
        return ms.agg_sum_grouped(gid, m1p, 1000), ms.agg_sum_grouped(gid, m2p, 1000)

    def chain_fused():  # the measured path of D-16: the semi-join fused (K7)
        pos1 = ms.select(k0, ms.BETWEEN, 0, 365, out_fmt=ms.delta_bp(512))
        pos2 = ms.semijoin(k1, pos1, bm, Dm[1])
        m1p = ms.project(m1, pos2, 0, ms.dyn_bp(512))
        m2p = ms.project(m2, pos2, 0, ms.dyn_bp(512))
        k3p = ms.project(k3, pos2, 0, ms.static_bp(17))
        gid = ms.project(gattr, k3p, 0, ms.static_bp(10))
        return ms.agg_sum_grouped(gid, m1p, 1000), ms.agg_sum_grouped(gid, m2p, 1000)

    alg = k0.footprint() + k1.footprint() + m1.footprint() + m2.footprint() + k3.footprint()
    report("c4", "full chain, fused semi-join K7 (select, semi-join, projects, grouped sums)",
           timed(chain_fused, reps), n, alg)
    report("c4", "full chain, operator at a time (select, project, select, project, ...)", timed(chain, reps), n,
           alg)
    pos1 = ms.select(k0, ms.BETWEEN, 0, 365, out_fmt=ms.delta_bp(512))
    report("c4", "select k0 in [0,365) -> DELTA_BP{512}",
           timed(lambda: ms.select(k0, ms.BETWEEN, 0, 365, out_fmt=ms.delta_bp(512)), reps), n,
           k0.footprint() + pos1.footprint())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--configs", default="c1,c2,c3,c4")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for c in a.configs.split(","):
        globals()[c](a.reps)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
