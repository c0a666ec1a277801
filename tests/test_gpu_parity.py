"""GPU parity: the CUDA path (through the C ABI) against the oracle, bit-exact
on every image section, on seeded inputs spanning several 2048-row tiles, a
ragged tail and the edge cases (empty, one value, block +-1, all-zero, 64-bit
values, wrap-around deltas)."""
import numpy as np
import pytest

import oracle as O
from tests.gpu_util import (assert_same_image, get_ms, oracle_fmt, oracle_op, rand_values, to_torch)

pytestmark = pytest.mark.gpu

LENGTHS = [0, 1, 127, 128, 129, 2047, 2048, 2049, 3 * 2048 + 7, 70_001]
KINDS = ["small", "wide", "sorted", "runs", "outlier", "zeros"]


def all_fmts():
    ms = get_ms()
    f = [ms.uncompr(), ms.static_bp(0), ms.static_bp(64), ms.rle()]
    for B in (128, 256, 512, 1024, 2048):
        f += [ms.dyn_bp(B), ms.for_bp(B), ms.delta_bp(B)]
    return f


@pytest.fixture(scope="module")
def rng():
    return np.random.default_rng(2024)


@pytest.mark.parametrize("kind", KINDS)
def test_compress_decompress(kind, rng):
    ms = get_ms()
    for n in LENGTHS:
        v = rand_values(n, kind, rng)
        t = to_torch(v)
        for f in all_fmts():
            oc = O.encode(v, *oracle_fmt(f))
            gc = ms.compress(t, f)
            assert_same_image(gc, oc, f"compress {f} {kind} n={n}")
            back = ms.to_u64_numpy(ms.decompress(gc)) if n else np.zeros(0, np.uint64)
            assert np.array_equal(back, v), f"decompress {f} {kind} n={n}"


def test_static_explicit_widths(rng):
    ms = get_ms()
    for w in (1, 3, 7, 10, 13, 20, 31, 32, 33, 40, 63):
        v = rng.integers(0, 1 << w, 5000, dtype=np.uint64)
        gc = ms.compress(to_torch(v), ms.static_bp(w))
        assert_same_image(gc, O.encode(v, O.STATIC_BP, w), f"static w={w}")
        assert np.array_equal(ms.to_u64_numpy(ms.decompress(gc)), v)


def test_width_overflow(rng):
    ms = get_ms()
    v = np.array([1, 2, 1 << 12], np.uint64)
    with pytest.raises(ms.MsError) as e:
        ms.compress(to_torch(v), ms.static_bp(8))
    assert e.value.code == 2  # MS_E_WIDTH_OVERFLOW


def test_invalid_descriptors():
    ms = get_ms()
    with pytest.raises(ms.MsError):
        ms.compress(to_torch(np.arange(10, dtype=np.uint64)), ms.Fmt(ms.DYN_BP, 0, 100))
    with pytest.raises(ms.MsError):
        ms.compress(to_torch(np.arange(10, dtype=np.uint64)), ms.Fmt(9, 0, 0))


@pytest.mark.parametrize("kind", ["small", "sorted", "runs", "outlier"])
def test_morph_pairs(kind, rng):
    ms = get_ms()
    fm = [ms.uncompr(), ms.static_bp(0), ms.dyn_bp(512), ms.for_bp(256), ms.delta_bp(2048), ms.delta_bp(128),
          ms.rle()]
    for n in (0, 2049, 3 * 2048 + 7, 50_000):
        v = rand_values(n, kind, rng)
        t = to_torch(v)
        for a in fm:
            ga = ms.compress(t, a)
            oa = O.encode(v, *oracle_fmt(a))
            for b in fm:
                gm = ms.morph(ga, b)
                assert_same_image(gm, O.morph(oa, *oracle_fmt(b)), f"morph {a}->{b} {kind} n={n}")


@pytest.mark.parametrize("case", ["far", "near", "wrap", "zeros"])
def test_morph_delta_to_static_auto_width(case):
    """DELTA_BP -> STATIC_BP{auto}: the width comes from the block headers when the
    bounds [max ref, max ref + (B-1)(2^w - 1)] share one effective width, else from a
    max pass over the decoded values; both give the oracle's image (P:122 width of
    the maximum). 'near': the maximum sits just under 2^30 so the bounds straddle it;
    'wrap': differences that wrap mod 2^64 (no header bound)."""
    ms = get_ms()
    rng = np.random.default_rng(3)
    n = 5 * 2048 + 77
    if case == "far":
        v = np.cumsum(rng.integers(0, 3, n)).astype(np.uint64) + np.uint64(1 << 29)
    elif case == "near":
        v = np.cumsum(rng.integers(0, 3, n)).astype(np.uint64)
        v = v + np.uint64((1 << 30) - 5 - int(v[-1]))
    elif case == "wrap":
        v = rng.integers(0, 1 << 40, n).astype(np.uint64)
    else:
        v = np.zeros(n, np.uint64)
    d = ms.compress(to_torch(v), ms.delta_bp(2048))
    ms.profile_read()
    ms.profile_enable(True)
    try:
        got = ms.morph(d, ms.static_bp(0))
        names = set(ms.profile_read())
    finally:
        ms.profile_enable(False)
    assert_same_image(got, O.morph(O.encode(v, O.DELTA_BP, 0, 2048), O.STATIC_BP, 0, 0), f"auto width {case}")
    assert ("delta_max" in names) == (case in ("near", "wrap")), names


@pytest.mark.parametrize("kind", ["small", "sorted", "runs", "outlier", "wide"])
def test_many_tiles_per_cta(kind, rng):
    """More 2048-row tiles than resident CTAs (148 SMs x 4): the staged engine's
    double-buffered pipeline runs several iterations per CTA, with a ragged tail."""
    ms = get_ms()
    n = (1 << 21) + 12_345
    v = rand_values(n, kind, rng)
    t = to_torch(v)
    fm = [ms.static_bp(0), ms.dyn_bp(512), ms.for_bp(128), ms.delta_bp(2048), ms.delta_bp(256), ms.rle()]
    for a in fm:
        oa = O.encode(v, *oracle_fmt(a))
        ga = ms.compress(t, a)
        assert_same_image(ga, oa, f"compress {a} {kind} n={n}")
        assert np.array_equal(ms.to_u64_numpy(ms.decompress(ga)), v), f"decompress {a} {kind}"
        for b in (ms.static_bp(0), ms.delta_bp(512), ms.for_bp(2048), ms.uncompr()):
            assert_same_image(ms.morph(ga, b), O.morph(oa, *oracle_fmt(b)), f"morph {a}->{b} {kind} n={n}")


PREDS = None


def preds(v):
    ms = get_ms()
    lo = int(np.sort(v)[len(v) // 3]) if len(v) else 5
    return [(ms.EQ, lo, 0), (ms.NE, lo, 0), (ms.LT, lo, 0), (ms.LE, lo, 0), (ms.GT, lo, 0), (ms.GE, lo, 0),
            (ms.BETWEEN, lo, lo + 40), (ms.LT, 0, 0), (ms.GE, 0, 0), (ms.GT, 2**64 - 1, 0),
            (ms.EQ, 2**64 - 1, 0)]


@pytest.mark.parametrize("kind", ["small", "sorted", "runs", "outlier", "wide"])
def test_select(kind, rng):
    ms = get_ms()
    in_fmts = [ms.uncompr(), ms.static_bp(0), ms.dyn_bp(512), ms.for_bp(128), ms.delta_bp(2048), ms.rle()]
    out_fmts = [ms.delta_bp(512), ms.uncompr(), ms.for_bp(128), ms.dyn_bp(2048), ms.static_bp(0),
                ms.static_bp(40), ms.rle(), ms.delta_bp(128)]
    for n in (1, 2049, 3 * 2048 + 7, 100_003):
        v = rand_values(n, kind, rng)
        t = to_torch(v)
        for fi in in_fmts:
            gi = ms.compress(t, fi)
            oi = O.encode(v, *oracle_fmt(fi))
            for op, a, b in preds(v):
                for fo in out_fmts:
                    for off in (0, 5_000_000_000):
                        gs = ms.select(gi, op, a, b, row_offset=off, out_fmt=fo)
                        os_ = O.select(oi, oracle_op(op), a, b, row_offset=off, out_fmt=oracle_fmt(fo)[0],
                                       out_width=fo.bit_width, out_block=fo.block_size)
                        assert_same_image(gs, os_, f"select {fi} {op} {a} -> {fo} {kind} n={n} off={off}")


def test_select_bitmap(rng):
    ms = get_ms()
    import torch
    bits = 200_000
    words = rng.integers(0, 2**64 - 1, (bits + 63) // 64, dtype=np.uint64, endpoint=True)
    words &= rng.integers(0, 2**64 - 1, words.size, dtype=np.uint64, endpoint=True)  # ~25% set
    bm = to_torch(words)
    v = rng.integers(0, 210_000, 70_000).astype(np.uint64)
    for fi in (ms.static_bp(18), ms.uncompr(), ms.dyn_bp(512)):
        gi = ms.compress(to_torch(v), fi)
        oi = O.encode(v, *oracle_fmt(fi))
        gs = ms.select(gi, ms.IN_BITMAP, bitmap=bm, bitmap_bits=bits, out_fmt=ms.delta_bp(512))
        os_ = O.select(oi, O.IN_BITMAP, bitmap=words, bitmap_bits=bits, out_fmt=O.DELTA_BP, out_block=512)
        assert_same_image(gs, os_, f"bitmap select {fi}")


@pytest.mark.parametrize("kind", ["small", "wide", "sorted", "runs"])
def test_project(kind, rng):
    ms = get_ms()
    n = 3 * 2048 + 77
    v = rand_values(n, kind, rng)
    t = to_torch(v)
    off = 1000
    sorted_pos = np.sort(rng.choice(n, 2500, replace=False)).astype(np.uint64) + np.uint64(off)
    unsorted_pos = rng.integers(0, n, 3000).astype(np.uint64) + np.uint64(off)
    data_fmts = [ms.uncompr(), ms.static_bp(0), ms.dyn_bp(512), ms.for_bp(512), ms.delta_bp(128), ms.rle()]
    pos_fmts = [ms.delta_bp(512), ms.uncompr(), ms.static_bp(0), ms.rle()]
    out_fmts = [ms.for_bp(512), ms.uncompr(), ms.dyn_bp(128), ms.static_bp(0), ms.delta_bp(512)]
    for fd in data_fmts:
        gd = ms.compress(t, fd)
        od = O.encode(v, *oracle_fmt(fd))
        for pos in (sorted_pos, unsorted_pos):
            for fp in pos_fmts:
                if fp.format == ms.RLE and pos is unsorted_pos:
                    continue
                gp = ms.compress(to_torch(pos), fp)
                op_ = O.encode(pos, *oracle_fmt(fp))
                for fo in out_fmts:
                    gr = ms.project(gd, gp, off, fo)
                    orr = O.project(od, op_, off, *oracle_fmt(fo))
                    assert_same_image(gr, orr, f"project {fd} @ {fp} -> {fo} {kind}")


@pytest.mark.parametrize("density", [3000, 9000])
def test_project_sequential_data_gather(rng, density):
    """DELTA_BP / RLE data gathered tile by tile (no whole-column decode, DP3),
    sparse and dense positions."""
    ms = get_ms()
    n = 5 * 2048 + 13
    v = rand_values(n, "sorted", rng)
    t = to_torch(v)
    pos = np.sort(rng.choice(n, density, replace=False)).astype(np.uint64)
    for fd in (ms.delta_bp(128), ms.delta_bp(2048), ms.rle()):
        gd = ms.compress(t, fd)
        od = O.encode(v, *oracle_fmt(fd))
        for fp in (ms.delta_bp(512), ms.uncompr()):
            gp = ms.compress(to_torch(pos), fp)
            op_ = O.encode(pos, *oracle_fmt(fp))
            for fo in (ms.delta_bp(512), ms.uncompr(), ms.for_bp(128)):
                assert_same_image(ms.project(gd, gp, 0, fo), O.project(od, op_, 0, *oracle_fmt(fo)),
                                  f"project {fd} @ {fp} -> {fo} (tiled)")


def test_project_range_error(rng):
    ms = get_ms()
    d = ms.compress(to_torch(np.arange(100, dtype=np.uint64)), ms.for_bp(128))
    p = ms.compress(to_torch(np.array([5, 100], np.uint64)), ms.uncompr())
    with pytest.raises(ms.MsError) as e:
        ms.project(d, p, 0, ms.uncompr())
    assert e.value.code == 4  # MS_E_RANGE


@pytest.mark.parametrize("kind", KINDS)
def test_agg_sum(kind, rng):
    ms = get_ms()
    for n in (0, 1, 2049, 3 * 512 + 11, 100_001):
        v = rand_values(n, kind, rng)
        t = to_torch(v)
        expect = O.agg_sum(O.encode(v, O.UNCOMPR))
        for f in all_fmts():
            g = ms.compress(t, f)
            assert ms.u64(ms.agg_sum(g)) == expect, f"sum {f} {kind} n={n}"
        if n:
            pos = np.sort(rng.choice(n, max(1, n // 3), replace=False)).astype(np.uint64) + np.uint64(7)
            ep = O.agg_sum(O.encode(v, O.UNCOMPR), O.encode(pos, O.UNCOMPR), 7)
            for fd in (ms.for_bp(512), ms.static_bp(0), ms.delta_bp(512), ms.rle(), ms.dyn_bp(128)):
                for fp in (ms.delta_bp(512), ms.uncompr(), ms.rle()):
                    g = ms.agg_sum(ms.compress(t, fd), ms.compress(to_torch(pos), fp), 7)
                    assert ms.u64(g) == ep, f"sum_at {fd} {fp} {kind} n={n}"
    ms.check_errors()


def test_agg_sum_grouped(rng):
    ms = get_ms()
    for n_groups in (7, 1000, 5000):
        n = 50_000
        g = rng.integers(0, n_groups, n).astype(np.uint64)
        v = rand_values(n, "wide", rng)
        expect = O.agg_sum_grouped(O.encode(g, O.UNCOMPR), O.encode(v, O.UNCOMPR), n_groups)
        for fg in (ms.uncompr(), ms.static_bp(0), ms.dyn_bp(512)):
            for fv in (ms.dyn_bp(512), ms.uncompr(), ms.for_bp(128)):
                out = ms.agg_sum_grouped(ms.compress(to_torch(g), fg), ms.compress(to_torch(v), fv), n_groups)
                assert np.array_equal(ms.to_u64_numpy(out), expect), (n_groups, fg, fv)
    ms.check_errors()
    bad = ms.compress(to_torch(np.array([1, 2, 9], np.uint64)), ms.uncompr())
    vals = ms.compress(to_torch(np.array([1, 2, 3], np.uint64)), ms.uncompr())
    ms.agg_sum_grouped(bad, vals, 5)
    with pytest.raises(ms.MsError) as e:
        ms.check_errors()
    assert e.value.code == 4


def test_host_roundtrip(rng):
    ms = get_ms()
    v = rand_values(10_000, "outlier", rng)
    oc = O.encode(v, O.FOR_BP, 0, 512)
    g = ms.Column.from_host(ms.for_bp(512), oc.n, oc.payload, oc.cw, oc.ref, oc.rem)
    assert_same_image(g, oc, "from_host")
    assert np.array_equal(ms.to_u64_numpy(ms.decompress(g)), v)


def test_select_dense_and_sparse(rng):
    """Width-1 deltas (every row selected), single matches, matches only in the
    remainder, and empty results, through every output format."""
    ms = get_ms()
    outs = [ms.delta_bp(512), ms.delta_bp(128), ms.delta_bp(2048), ms.for_bp(512), ms.dyn_bp(1024),
            ms.uncompr(), ms.static_bp(0), ms.rle()]
    cases = []
    n = 100_003
    z = np.zeros(n, np.uint64)
    cases.append((z, ms.GE, 0, 0))                       # all rows
    one = z.copy(); one[77_777] = 5
    cases.append((one, ms.EQ, 5, 0))                      # a single match
    tail = z.copy(); tail[-3:] = 9
    cases.append((tail, ms.EQ, 9, 0))                     # matches only in the final rows
    cases.append((z, ms.EQ, 1, 0))                        # nothing
    sparse = rng.integers(0, 1 << 20, n).astype(np.uint64)
    cases.append((sparse, ms.LT, 1 << 8, 0))             # ~0.02% selectivity
    for v, op, a, b in cases:
        for fi in (ms.dyn_bp(512), ms.static_bp(0), ms.uncompr()):
            gi = ms.compress(to_torch(v), fi)
            oi = O.encode(v, *oracle_fmt(fi))
            for fo in outs:
                gs = ms.select(gi, op, a, b, row_offset=3, out_fmt=fo)
                os_ = O.select(oi, oracle_op(op), a, b, row_offset=3, out_fmt=oracle_fmt(fo)[0],
                               out_width=fo.bit_width, out_block=fo.block_size)
                assert_same_image(gs, os_, f"select dense/sparse {fi} {op} {a} -> {fo}")


def test_max_width_hint(rng):
    """The descriptor's max_width sizing hint is set by producers; a wrong hint
    costs speed, never correctness: chunks wider than the staging stage it sized
    are read from global memory (selstream.cuh), and the result is exact."""
    ms = get_ms()
    v = rng.integers(0, 1 << 20, 10_000).astype(np.uint64)
    v[5000] = (1 << 40) + 3
    c = ms.compress(to_torch(v), ms.dyn_bp(512))
    w = np.diff(O.encode(v, O.DYN_BP, 0, 512).cw.astype(np.int64))
    assert c.max_width == int(w.max()) == 41
    narrow = ms.compress(to_torch(v & np.uint64(0xFFFFF)), ms.dyn_bp(512))
    assert narrow.max_width == 20
    # a hint that understates the widths of two adjacent wide blocks (their chunk
    # overruns a stage sized for 20 bits): read from global memory, exact
    v2 = v.copy()
    v2[512 * 4 + 7] = (1 << 40) + 1
    v2[512 * 5 + 9] = (1 << 40) + 2
    c2 = ms.compress(to_torch(v2), ms.dyn_bp(512))
    c2._c.fmt.max_width = 20
    gs2 = ms.select(c2, ms.LT, 1 << 16, out_fmt=ms.delta_bp(512))
    assert_same_image(gs2, O.select(O.encode(v2, O.DYN_BP, 0, 512), O.LT, 1 << 16, out_fmt=O.DELTA_BP,
                                    out_block=512), "select with an understated hint (unstaged chunk)")
    assert ms.u64(ms.agg_sum(c2)) == int(v2.sum(dtype=np.uint64))
    # a hint that is wrong but harmless still gives the exact result
    c._c.fmt.max_width = 20
    gs = ms.select(c, ms.LT, 1 << 16, out_fmt=ms.delta_bp(512))
    assert_same_image(gs, O.select(O.encode(v, O.DYN_BP, 0, 512), O.LT, 1 << 16, out_fmt=O.DELTA_BP,
                                   out_block=512), "select with understated hint")


@pytest.mark.parametrize("fname", ["dyn1024", "for2048", "static", "dyn512"])
def test_select_stream_many_chunks(fname, rng):
    """The CTA-streamed select / sum core (selstream.cuh) over more chunks per CTA
    than stages (16 segments per chunk, 10 stages, 148 CTAs: > 12M rows), blocks
    larger than a segment (B = 1024, 2048: segments inside a block), a static
    width, a ragged tail of partial segments and the block remainder; images and
    sums against the oracle."""
    ms = get_ms()
    n = (1 << 24) + 12_345
    v = rng.integers(0, 1 << 19, n).astype(np.uint64)
    v[rng.random(n) < 0.001] = np.uint64(1 << 21)  # some wider blocks
    f = {"dyn1024": ms.dyn_bp(1024), "for2048": ms.for_bp(2048), "static": ms.static_bp(0),
         "dyn512": ms.dyn_bp(512)}[fname]
    gi = ms.compress(to_torch(v), f)
    oi = O.encode(v, *oracle_fmt(f))
    ms.profile_read()
    ms.profile_enable(True)
    try:
        for op, a, b in ((ms.LT, 1 << 15, 0), (ms.BETWEEN, 1000, 1 << 18)):
            gs = ms.select(gi, op, a, b, out_fmt=ms.delta_bp(512))
            os_ = O.select(oi, oracle_op(op), a, b, out_fmt=O.DELTA_BP, out_block=512)
            assert_same_image(gs, os_, f"select {f} {op}")
        assert ms.u64(ms.agg_sum(gi)) == int(v.sum(dtype=np.uint64))
        names = set(ms.profile_read())
    finally:
        ms.profile_enable(False)
    assert "select_stream" in names and "sum_stream" in names, names


@pytest.mark.parametrize("kind", ["small", "sorted", "wide"])
def test_compress_stream_stage_reuse(kind, rng):
    """u64 -> DYN / FOR / DELTA_BP through the streamed compress (cstream.cuh) with
    more 2048-row tiles per CTA than its 13 stages, every block size, a ragged
    tail; byte-exact against the oracle."""
    ms = get_ms()
    n = (1 << 23) + 77
    v = rand_values(n, kind, rng)
    t = to_torch(v)
    ms.profile_read()
    ms.profile_enable(True)
    try:
        for f in (ms.dyn_bp(128), ms.for_bp(512), ms.delta_bp(2048), ms.delta_bp(256), ms.for_bp(1024)):
            assert_same_image(ms.compress(t, f), O.encode(v, *oracle_fmt(f)), f"compress {f} {kind}")
        names = set(ms.profile_read())
    finally:
        ms.profile_enable(False)
    assert "compress_stream" in names


@pytest.mark.parametrize("kind", ["values", "steps"])
def test_compress_stream_narrow_and_wide_tiles(kind, rng):
    """cstream.cuh picks its packer per 2048-row tile: the staged u32 packer when every
    block of the tile is <= 16 bits wide, the word builder otherwise. Narrow values (or
    steps) with rare 40-bit outliers mix both kinds of tile, and widths that differ
    between the blocks of one tile, in one column; bases near a multiple of 2^32 make
    the staged packer's low-word differences wrap. Byte-exact against the oracle."""
    ms = get_ms()
    n = (1 << 22) + 5
    x = rng.integers(0, 1 << 10, n).astype(np.uint64)
    x[(np.arange(n) >> 7) % 3 == 0] &= np.uint64(3)  # every third 128-row stretch narrower: widths differ inside a tile
    hit = rng.random(n) < 1e-4                  # ~0.2 outliers per 2048-row tile
    x[hit] = (np.uint64(1) << np.uint64(40)) + x[hit]
    if kind == "values":
        v = x + np.uint64((1 << 32) - 300)       # FOR: min just below 2^32, values across it
    else:
        v = np.cumsum(x, dtype=np.uint64) + np.uint64((1 << 32) - 5000)  # DELTA: narrow steps, rare wide ones
    t = to_torch(v)
    ms.profile_read()
    ms.profile_enable(True)
    try:
        for f in (ms.dyn_bp(128), ms.for_bp(128), ms.for_bp(512), ms.delta_bp(256), ms.delta_bp(2048)):
            g = ms.compress(t, f)
            assert_same_image(g, O.encode(v, *oracle_fmt(f)), f"compress {f} {kind}")
            assert np.array_equal(ms.to_u64_numpy(ms.decompress(g)), v)
        names = set(ms.profile_read())
    finally:
        ms.profile_enable(False)
    assert "compress_stream" in names
