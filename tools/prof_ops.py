#!/usr/bin/env python3
"""Per-kernel CUDA-event times (libms's own profiling) of single ops of the
BASELINE configs, to see which launch of a multi-kernel op dominates.
usage: python tools/prof_ops.py [c3|c4|c2]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2004_09350_b200 import ms  # noqa: E402


def prof(name, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ms.profile_read()
    ms.profile_enable(True)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    ms.profile_enable(False)
    p = ms.profile_read()
    tot = sum(t for _, t in p.values()) / reps
    print(f"{name}: {tot:.3f} ms in kernels | " + ", ".join(f"{k}={t / reps:.3f}" for k, (c, t) in
                                                        sorted(p.items(), key=lambda kv: -kv[1][1])), flush=True)


def c3():
    n = 1 << 29
    x = synth.gen_torch("c3.x", n)
    R = ms.compress(x, ms.rle())
    D = ms.compress(x, ms.delta_bp(2048))
    prof("compress DELTA_BP{2048}", lambda: ms.compress(x, ms.delta_bp(2048)))
    prof("compress RLE", lambda: ms.compress(x, ms.rle()))
    del x
    prof("morph RLE -> DELTA_BP{2048}", lambda: ms.morph(R, ms.delta_bp(2048)))
    prof("morph DELTA -> STATIC auto", lambda: ms.morph(D, ms.static_bp(0)))
    prof("select DELTA", lambda: ms.select(D, ms.BETWEEN, 10**6, 2 * 10**6, out_fmt=ms.delta_bp(512)))
    prof("select RLE", lambda: ms.select(R, ms.BETWEEN, 10**6, 2 * 10**6, out_fmt=ms.delta_bp(512)))


def c3e():  # the engine ops of c3 only (for ncu: -k regex:engine_kernel)
    n = 1 << 29
    x = synth.gen_torch("c3.x", n)
    D = ms.compress(x, ms.delta_bp(2048))
    prof("compress DELTA_BP{2048}", lambda: ms.compress(x, ms.delta_bp(2048)), reps=1)
    del x
    prof("morph DELTA -> STATIC auto", lambda: ms.morph(D, ms.static_bp(0)), reps=1)
    prof("decompress DELTA", lambda: ms.decompress(D), reps=1)
    R = ms.morph(D, ms.rle())
    prof("decompress RLE", lambda: ms.decompress(R), reps=1)
    prof("morph RLE -> DYN_BP{512}", lambda: ms.morph(R, ms.dyn_bp(512)), reps=1)


def c2e():  # compress of c2's X (UNCOMPR -> DYN_BP{512}) only (for ncu: -k regex:engine_kernel)
    n = 1 << 28
    x = synth.gen_torch("c2.X", n)
    prof("compress c2.X -> DYN_BP{512}", lambda: ms.compress(x, ms.dyn_bp(512)), reps=1)
    prof("compress c2.X -> FOR_BP{512}", lambda: ms.compress(x, ms.for_bp(512)), reps=1)
    prof("compress c2.X -> STATIC_BP{auto}", lambda: ms.compress(x, ms.static_bp(0)), reps=1)


def c4():
    n = 600_000_000
    Dm = synth.D4
    bm = torch.from_numpy(synth.bitmap_c4().view("int64")).cuda()
    gattr = ms.compress(synth.gen_torch("c4.gattr", Dm[3]), ms.static_bp(10))
    k0 = ms.compress(synth.gen_torch("c4.k0", n), ms.static_bp(12))
    k1 = ms.compress(synth.gen_torch("c4.k1", n), ms.static_bp(18))
    k3 = ms.compress(synth.gen_torch("c4.k3", n), ms.static_bp(17))
    m1 = ms.compress(synth.gen_torch("c4.m1", n), ms.dyn_bp(512))
    pos1 = ms.select(k0, ms.BETWEEN, 0, 365, out_fmt=ms.delta_bp(512))
    prof("select k0", lambda: ms.select(k0, ms.BETWEEN, 0, 365, out_fmt=ms.delta_bp(512)))
    prof("project k1 -> STATIC 18", lambda: ms.project(k1, pos1, 0, ms.static_bp(18)))
    k1p = ms.project(k1, pos1, 0, ms.static_bp(18))
    prof("select k1' IN_BITMAP", lambda: ms.select(k1p, ms.IN_BITMAP, bitmap=bm, bitmap_bits=Dm[1],
                                                    out_fmt=ms.delta_bp(512)))
    idx = ms.select(k1p, ms.IN_BITMAP, bitmap=bm, bitmap_bits=Dm[1], out_fmt=ms.delta_bp(512))
    prof("project pos1 @ idx -> DELTA", lambda: ms.project(pos1, idx, 0, ms.delta_bp(512)))
    pos2 = ms.project(pos1, idx, 0, ms.delta_bp(512))
    prof("project m1 -> DYN", lambda: ms.project(m1, pos2, 0, ms.dyn_bp(512)))
    m1p = ms.project(m1, pos2, 0, ms.dyn_bp(512))
    prof("project k3 -> STATIC 17", lambda: ms.project(k3, pos2, 0, ms.static_bp(17)))
    k3p = ms.project(k3, pos2, 0, ms.static_bp(17))
    prof("project gattr @ k3' -> STATIC 10", lambda: ms.project(gattr, k3p, 0, ms.static_bp(10)))
    gid = ms.project(gattr, k3p, 0, ms.static_bp(10))
    prof("grouped sum", lambda: ms.agg_sum_grouped(gid, m1p, 1000))


def c4f():  # the fused D-16 chain (K7 semi-join), operator by operator
    n = 600_000_000
    Dm = synth.D4
    bm = torch.from_numpy(synth.bitmap_c4().view("int64")).cuda()
    gattr = ms.compress(synth.gen_torch("c4.gattr", Dm[3]), ms.static_bp(10))
    k0 = ms.compress(synth.gen_torch("c4.k0", n), ms.static_bp(12))
    k1 = ms.compress(synth.gen_torch("c4.k1", n), ms.static_bp(18))
    k3 = ms.compress(synth.gen_torch("c4.k3", n), ms.static_bp(17))
    m1 = ms.compress(synth.gen_torch("c4.m1", n), ms.dyn_bp(512))
    pos1 = ms.select(k0, ms.BETWEEN, 0, 365, out_fmt=ms.delta_bp(512))
    prof("select k0", lambda: ms.select(k0, ms.BETWEEN, 0, 365, out_fmt=ms.delta_bp(512)))
    pos2 = ms.semijoin(k1, pos1, bm, Dm[1])
    prof("semijoin k1 @ pos1", lambda: ms.semijoin(k1, pos1, bm, Dm[1]))
    prof("project m1 @ pos2 -> DYN", lambda: ms.project(m1, pos2, 0, ms.dyn_bp(512)))
    k3p = ms.project(k3, pos2, 0, ms.static_bp(17))
    prof("project k3 @ pos2 -> STATIC 17", lambda: ms.project(k3, pos2, 0, ms.static_bp(17)))
    gid = ms.project(gattr, k3p, 0, ms.static_bp(10))
    prof("project gattr @ k3' -> STATIC 10", lambda: ms.project(gattr, k3p, 0, ms.static_bp(10)))
    m1p = ms.project(m1, pos2, 0, ms.dyn_bp(512))
    prof("grouped sum", lambda: ms.agg_sum_grouped(gid, m1p, 1000))
    print(f"pos1 {pos1.n} pos2 {pos2.n}", flush=True)


def c2():
    n = 1 << 28
    X = ms.compress(synth.gen_torch("c2.X", n), ms.dyn_bp(512))
    prof("select c2", lambda: ms.select(X, ms.EQ, 17, out_fmt=ms.delta_bp(512)))


def sweep():
    import numpy as np
    n = 1 << 27
    v = synth.gen_host("C1.X", n)
    t = torch.from_numpy(v.view(np.int64)).cuda()
    X = ms.compress(t, ms.static_bp(0))
    for f, name in ((ms.uncompr(), "UNCOMPR"), (ms.delta_bp(512), "DELTA_BP512"), (ms.dyn_bp(512), "DYN_BP512")):
        prof(f"C1 static -> {name}", lambda: ms.select(X, ms.EQ, 0, out_fmt=f))


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for c in (sys.argv[1:] or ["c2", "c3", "c4"]):
        globals()[c]()
        torch.cuda.empty_cache()
