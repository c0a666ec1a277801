"""GPU parity of the plan-level operators (plan.cu)
against oracle/plan_ops.py, byte for byte: the exact-size format profile and the
choice it drives (every candidate's size equals the oracle's footprint of the
canonical image), intersect / merge of positions, equi-join, group ids and
extents, elementwise arithmetic — over every input format, ragged sizes and the
degenerate cases (empty inputs, disjoint ranges, duplicates, NotSorted)."""
import zlib

import numpy as np
import pytest

import oracle as O
import synth
from oracle import plan_ops as P
from tests.gpu_util import assert_same_image, get_ms, oracle_fmt, rand_values, to_torch

pytestmark = pytest.mark.gpu


@pytest.fixture
def rng(request):
    return np.random.default_rng(zlib.crc32(request.node.name.encode()))


def fmt_of(ms, name):
    return {"uncompr": ms.uncompr(), "static": ms.static_bp(0), "dyn512": ms.dyn_bp(512),
            "for128": ms.for_bp(128), "delta2048": ms.delta_bp(2048), "rle": ms.rle(),
            "delta512": ms.delta_bp(512)}[name]


def col(ms, v, name):
    return ms.compress(to_torch(np.ascontiguousarray(v, np.uint64)), fmt_of(ms, name))


@pytest.mark.parametrize("kind", ["small", "sorted", "runs", "outlier", "wide", "zeros"])
@pytest.mark.parametrize("B", [128, 512, 2048])
def test_format_sizes_exact(kind, B, rng):
    ms = get_ms()
    for n in (0, 1, B - 1, B, 3 * 2048 + 77, 70_001):
        v = rand_values(n, kind, rng)
        for fi in ("uncompr", "dyn512", "rle"):
            sizes, best = ms.format_sizes(col(ms, v, fi), B)
            want = P.format_sizes(v, B)
            assert [sizes[k] for k in ms.CANDIDATES] == want, (kind, B, n, fi)
            assert best.format == P.choose_format(v, B)


@pytest.mark.parametrize("c", ["C1.plain", "C2.plain", "C3.Y", "C4.Y"])
def test_choose_format_paper_columns(c):
    """P:577-582's best formats per column on the footprint objective, from the GPU."""
    ms = get_ms()
    v = synth.gen_host(c, 1 << 18)
    _, best = ms.format_sizes(col(ms, v, "uncompr"), 512)
    assert best.format == P.choose_format(v, 512)


def sorted_positions(rng, n, universe, off=0):
    return (np.sort(rng.choice(universe, size=min(n, universe), replace=False)) + off).astype(np.uint64)


@pytest.mark.parametrize("fa,fb", [("delta512", "delta512"), ("uncompr", "delta2048"), ("rle", "static"),
                                   ("dyn512", "for128")])
def test_intersect_merge(fa, fb, rng):
    ms = get_ms()
    for na, nb, uni, off in ((5000, 7000, 60_000, 0), (40_000, 300, 1 << 22, 5_000_000_000), (1, 1, 3, 7),
                             (3000, 3000, 3000, 0)):
        a = sorted_positions(rng, na, uni, off)
        b = sorted_positions(rng, nb, uni, off)
        for fo in (ms.delta_bp(512), ms.uncompr(), ms.for_bp(128)):
            gi = ms.intersect(col(ms, a, fa), col(ms, b, fb), fo)
            gm = ms.merge(col(ms, a, fa), col(ms, b, fb), fo)
            assert_same_image(gi, O.encode(P.intersect_sorted(a, b), *oracle_fmt(fo)), f"intersect {fa} {fb} {fo}")
            assert_same_image(gm, O.encode(P.merge_sorted(a, b), *oracle_fmt(fo)), f"merge {fa} {fb} {fo}")


def test_intersect_merge_degenerate():
    ms = get_ms()
    a = np.array([1, 5, 9], np.uint64)
    e = np.zeros(0, np.uint64)
    far = np.array([100, 200], np.uint64)
    assert ms.intersect(col(ms, a, "uncompr"), col(ms, e, "uncompr"), ms.uncompr()).n == 0
    assert ms.intersect(col(ms, a, "uncompr"), col(ms, far, "uncompr"), ms.uncompr()).n == 0
    m = ms.merge(col(ms, a, "uncompr"), col(ms, e, "uncompr"), ms.uncompr())
    assert ms.to_u64_numpy(ms.decompress(m)).tolist() == [1, 5, 9]
    assert ms.merge(col(ms, e, "uncompr"), col(ms, e, "uncompr"), ms.delta_bp(512)).n == 0
    with pytest.raises(ms.MsError) as ex:  # NotSorted
        ms.intersect(col(ms, np.array([3, 2, 8], np.uint64), "uncompr"), col(ms, a, "uncompr"), ms.uncompr())
    assert ex.value.code == 1


@pytest.mark.parametrize("fl,fr", [("uncompr", "uncompr"), ("static", "dyn512"), ("rle", "delta2048")])
def test_join(fl, fr, rng):
    ms = get_ms()
    cases = [
        (rng.integers(0, 50, 20_000), rng.permutation(50)),               # FK -> unique PK (SSB shape)
        (rng.integers(0, 40, 3000), rng.integers(0, 40, 5000)),           # duplicates on both sides
        (rng.integers(0, 10, 100), rng.integers(100, 200, 50)),           # disjoint
        (np.array([1, 2, 3]), np.array([2, 2, 4])),
        (rng.integers(0, 2**64 - 1, 3000, dtype=np.uint64, endpoint=True), None),
    ]
    for L, R in cases:
        L = np.asarray(L, np.uint64)
        R = L[::-3].copy() if R is None else np.asarray(R, np.uint64)
        gl, gr = ms.join(col(ms, L, fl), col(ms, R, fr), ms.delta_bp(512) if R.size <= L.size else ms.uncompr(),
                         ms.uncompr())
        ol, orr = P.join_eq(L, R)
        assert np.array_equal(ms.to_u64_numpy(ms.decompress(gl)), ol), (fl, fr, L.size, R.size)
        assert np.array_equal(ms.to_u64_numpy(ms.decompress(gr)), orr), (fl, fr, L.size, R.size)


@pytest.mark.parametrize("fk", ["uncompr", "dyn512", "rle", "static"])
def test_group(fk, rng):
    ms = get_ms()
    for n, card in ((1, 1), (5000, 7), (70_001, 3000), (3 * 2048 + 5, 3 * 2048 + 5)):
        keys = rng.integers(0, card, n).astype(np.uint64)
        ids, ext = ms.group(col(ms, keys, fk), ids_fmt=ms.dyn_bp(512), extents_fmt=ms.uncompr())
        oid, oext = P.group(keys)
        assert_same_image(ids, O.encode(oid, O.DYN_BP, 0, 512), f"group ids {fk} n={n}")
        assert_same_image(ext, O.encode(oext, O.UNCOMPR), f"group extents {fk} n={n}")
        # refinement by a second key (prev ids = the first grouping)
        keys2 = rng.integers(0, 3, n).astype(np.uint64)
        ids2, ext2 = ms.group(col(ms, keys2, fk), prev_ids=ids, extents_fmt=ms.delta_bp(512))
        oid2, oext2 = P.group(keys2, oid)
        assert np.array_equal(ms.to_u64_numpy(ms.decompress(ids2)), oid2)
        assert_same_image(ext2, O.encode(oext2, O.DELTA_BP, 0, 512), f"group refine {fk} n={n}")
    with pytest.raises(ms.MsError):  # LengthMismatch
        ms.group(col(ms, np.arange(5, dtype=np.uint64), fk), prev_ids=col(ms, np.arange(4, dtype=np.uint64), fk))


@pytest.mark.parametrize("fa,fb", [("uncompr", "dyn512"), ("for128", "delta2048"), ("rle", "static")])
def test_calc(fa, fb, rng):
    ms = get_ms()
    for n in (0, 1, 3 * 2048 + 9, 50_000):
        a = rand_values(n, "wide", rng)
        b = rand_values(n, "small", rng)
        for op in (ms.ADD, ms.SUB, ms.MUL):
            for fo in (ms.uncompr(), ms.dyn_bp(512)):
                g = ms.calc(op, col(ms, a, fa), col(ms, b, fb), fo)
                assert_same_image(g, O.encode(P.calc_binary(op, a, b), *oracle_fmt(fo)), f"calc {op} {fa} {fb}")
    with pytest.raises(ms.MsError):
        ms.calc(ms.ADD, col(ms, np.arange(3, dtype=np.uint64), fa), col(ms, np.arange(4, dtype=np.uint64), fb))
