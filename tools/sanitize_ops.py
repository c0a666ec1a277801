#!/usr/bin/env python3
"""Small invocations of every libms entry point (all formats, select / project /
sum / grouped sum / morph / compress / decompress, error paths), checked against
the oracle — the workload for compute-sanitizer (memcheck, racecheck, synccheck,
initcheck): tools/sanitize.sh. Sizes span several tiles and ragged tails but stay
small so the instrumented run finishes in minutes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_2004_09350_b200 import ms  # noqa: E402


def t(v):
    return torch.from_numpy(np.ascontiguousarray(v, np.uint64).view(np.int64).copy()).cuda()


def code(f):
    return {ms.UNCOMPR: O.UNCOMPR, ms.STATIC_BP: O.STATIC_BP, ms.DYN_BP: O.DYN_BP, ms.DELTA_BP: O.DELTA_BP,
            ms.FOR_BP: O.FOR_BP, ms.RLE: O.RLE}[f.format], f.bit_width, f.block_size


def same(g, o, what):
    img = g.images()
    for s in ("payload", "cw", "ref", "rem"):
        assert np.array_equal(img[s], getattr(o, s)), (what, s)


def main():
    rng = np.random.default_rng(1)
    n = 3 * 2048 + 4097
    vals = {"small": rng.integers(0, 1000, n).astype(np.uint64),
            "sorted": np.sort(rng.integers(0, 1 << 30, n)).astype(np.uint64),
            "runs": np.repeat(rng.integers(0, 9, n // 5 + 1), 5)[:n].astype(np.uint64)}
    fmts = [ms.uncompr(), ms.static_bp(0), ms.dyn_bp(512), ms.for_bp(128), ms.delta_bp(2048), ms.rle()]
    outs = [ms.delta_bp(512), ms.uncompr(), ms.for_bp(128), ms.static_bp(0), ms.delta_bp(128), ms.rle()]
    checks = 0
    for kind, v in vals.items():
        tv = t(v)
        for f in fmts:
            g = ms.compress(tv, f)
            o = O.encode(v, *code(f))
            same(g, o, f"compress {f} {kind}")
            assert np.array_equal(ms.to_u64_numpy(ms.decompress(g)), v)
            thr = int(np.sort(v)[n // 3])
            for fo in outs:
                gs = ms.select(g, ms.LT, thr, row_offset=7, out_fmt=fo)
                os_ = O.select(o, O.LT, thr, row_offset=7, out_fmt=code(fo)[0], out_width=fo.bit_width,
                               out_block=fo.block_size)
                same(gs, os_, f"select {f}->{fo}")
                checks += 1
            pos = ms.select(g, ms.LT, thr, out_fmt=ms.delta_bp(512))
            opos = O.select(o, O.LT, thr, out_fmt=O.DELTA_BP, out_block=512)
            for fo in (ms.for_bp(512), ms.uncompr(), ms.dyn_bp(2048)):
                same(ms.project(g, pos, 0, fo), O.project(o, opos, 0, *code(fo)), f"project {f}->{fo}")
                checks += 1
            assert ms.u64(ms.agg_sum(g, check=True)) == O.agg_sum(o)
            assert ms.u64(ms.agg_sum(g, pos, check=True)) == O.agg_sum(o, opos)
            for fm in (ms.static_bp(0), ms.delta_bp(512), ms.rle(), ms.for_bp(2048)):
                same(ms.morph(g, fm), O.morph(o, *code(fm)), f"morph {f}->{fm}")
                checks += 1
    gid = rng.integers(0, 37, n).astype(np.uint64)
    gs = ms.to_u64_numpy(ms.agg_sum_grouped(ms.compress(t(gid), ms.static_bp(6)),
                                            ms.compress(t(vals["small"]), ms.dyn_bp(512)), 37, check=True))
    assert np.array_equal(gs, O.agg_sum_grouped(O.encode(gid, O.UNCOMPR), O.encode(vals["small"], O.UNCOMPR), 37))
    try:  # an error path: position out of range
        ms.project(ms.compress(tv, ms.for_bp(128)), ms.compress(t(np.array([n + 5], np.uint64)), ms.uncompr()))
        raise AssertionError("expected MS_E_RANGE")
    except ms.MsError as e:
        assert e.code == 4
    torch.cuda.synchronize()
    print(f"sanitize_ops ok: {checks} image checks, launches={ms.launch_count()}")


if __name__ == "__main__":
    main()
