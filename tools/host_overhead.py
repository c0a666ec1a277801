#!/usr/bin/env python3
"""Host-side cost of the c5 chain's operators: the step at a tiny size (2^20 rows,
kernels negligible) timed by wall clock per op, to see how much of the step's gap
between kernels is host work after each size read-back.
usage: python tools/host_overhead.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2004_09350_b200 import ms  # noqa: E402

n = 1 << 20
X = ms.compress(synth.gen_torch("c5.X", n), ms.dyn_bp(512))
Y = ms.compress(synth.gen_torch("c5.Y", n), ms.for_bp(512))
for _ in range(20):
    pos = ms.select(X, ms.LT, 1 << 16, out_fmt=ms.delta_bp(512))
    yp = ms.project(Y, pos, 0, ms.for_bp(512))
    s = ms.agg_sum(yp)
torch.cuda.synchronize()
R = 200
t = {"select": 0.0, "project": 0.0, "sum": 0.0}
t0 = time.perf_counter()
for _ in range(R):
    a = time.perf_counter()
    pos = ms.select(X, ms.LT, 1 << 16, out_fmt=ms.delta_bp(512))
    b = time.perf_counter()
    yp = ms.project(Y, pos, 0, ms.for_bp(512))
    c = time.perf_counter()
    s = ms.agg_sum(yp)
    torch.cuda.synchronize()
    d = time.perf_counter()
    t["select"] += b - a
    t["project"] += c - b
    t["sum"] += d - c
tot = time.perf_counter() - t0
print({k: round(v / R * 1e3, 4) for k, v in t.items()}, "ms per op; step", round(tot / R * 1e3, 4), "ms")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms.profile_read()
ms.profile_enable(True)
for _ in range(R):
    pos = ms.select(X, ms.LT, 1 << 16, out_fmt=ms.delta_bp(512))
    yp = ms.project(Y, pos, 0, ms.for_bp(512))
    s = ms.agg_sum(yp)
torch.cuda.synchronize()
ms.profile_enable(False)
p = ms.profile_read()
print("kernel ms per step:", round(sum(v[1] for v in p.values()) / R, 4), {k: round(v[1] / R, 4) for k, v in p.items()})
