"""Oracle pins: operators select / project / sum / grouped sum / morph
(SPEC.md S:257-363). Pinned by
SPEC's worked examples, brute-force numpy results, the RLE/FOR/DELTA sum
identities and the invariants S:339-342."""
import numpy as np
import pytest

import oracle as O
from tests.conftest import as_int
from tests.test_oracle_formats import rand_column

RNG = np.random.default_rng(7)
M64 = (1 << 64) - 1

FMTS = [(O.UNCOMPR, 0, 0), (O.STATIC_BP, 0, 0), (O.DYN_BP, 0, 128), (O.DYN_BP, 0, 512),
        (O.FOR_BP, 0, 512), (O.DELTA_BP, 0, 512), (O.DELTA_BP, 0, 2048), (O.RLE, 0, 0)]


def np_pred(v, op, a, b=0, bitmap=None, bits=0):
    v = v.astype(np.uint64)
    a, b = np.uint64(a), np.uint64(b)
    if op == O.EQ: return v == a
    if op == O.NE: return v != a
    if op == O.LT: return v < a
    if op == O.LE: return v <= a
    if op == O.GT: return v > a
    if op == O.GE: return v >= a
    if op == O.BETWEEN: return (v >= a) & (v < b)
    if op == O.IN_BITMAP:
        out = np.zeros(v.size, bool)
        inr = v < np.uint64(bits)
        idx = v[inr].astype(np.int64)
        out[inr] = ((bitmap[idx // 64] >> (idx % 64).astype(np.uint64)) & np.uint64(1)) == 1
        return out
    raise ValueError(op)


def test_select_worked_example(worked):
    ex = worked["select"]
    c = O.encode(ex["values"], O.UNCOMPR)
    out = O.select(c, O.EQ, ex["a"], out_fmt=O.UNCOMPR)
    assert list(O.decode(out)) == ex["positions"]


def test_project_worked_example(worked):
    ex = worked["project"]
    d = O.encode(ex["data"], O.UNCOMPR)
    p = O.encode(ex["positions"], O.UNCOMPR)
    assert list(O.decode(O.project(d, p))) == ex["expected"]


def test_sum_worked_examples(worked):
    assert O.agg_sum(O.encode(worked["sum"]["values"], O.UNCOMPR)) == worked["sum"]["expected"]
    ex = worked["sum_grouped"]
    g = O.agg_sum_grouped(O.encode(ex["gid"], O.UNCOMPR), O.encode(ex["values"], O.UNCOMPR), ex["n_groups"])
    assert list(g) == ex["expected"]
    ex = worked["sum_wrap"]
    assert O.agg_sum(O.encode([as_int(x) for x in ex["values"]], O.UNCOMPR)) == ex["expected"]


@pytest.mark.parametrize("kind", ["small", "sorted", "runs", "outlier"])
def test_select_brute_force_and_invariants(kind):
    n = 5000
    v = rand_column(n, kind)
    bitmap = RNG.integers(0, 2**63, 2, dtype=np.uint64)
    lo = int(np.sort(v)[n // 3])
    preds = [(O.EQ, lo, 0), (O.NE, lo, 0), (O.LT, lo, 0), (O.LE, lo, 0), (O.GT, lo, 0), (O.GE, lo, 0),
             (O.BETWEEN, lo, lo + 40), (O.LT, 0, 0), (O.GE, 0, 0), (O.IN_BITMAP, 0, 0)]
    for f, w, B in FMTS:
        col = O.encode(v, f, w, B)
        for op, a, b in preds:
            expect = np.nonzero(np_pred(v, op, a, b, bitmap, 128))[0].astype(np.uint64) + np.uint64(1000)
            for of, ow, oB in [(O.DELTA_BP, 0, 512), (O.UNCOMPR, 0, 0), (O.FOR_BP, 0, 128), (O.STATIC_BP, 0, 0)]:
                out = O.select(col, op, a, b, bitmap, 128, row_offset=1000, out_fmt=of, out_width=ow,
                               out_block=oB)
                got = O.decode(out)
                # format transparency: same positions for every in/out format
                assert np.array_equal(got, expect), (f, B, op, of)
            # invariants: strictly increasing and within [offset, offset+n)
            if got.size:
                assert (np.diff(got.astype(np.int64)) > 0).all() and got[-1] < 1000 + n


def test_select_saturated_predicates():
    # constants beyond the code range select all / nothing
    v = RNG.integers(0, 1 << 10, 3000).astype(np.uint64)
    c = O.encode(v, O.STATIC_BP, 10)
    assert O.select(c, O.LT, 1 << 40, out_fmt=O.UNCOMPR).n == 3000
    assert O.select(c, O.GE, 1 << 40, out_fmt=O.UNCOMPR).n == 0
    assert O.select(c, O.EQ, 1 << 10, out_fmt=O.UNCOMPR).n == 0


@pytest.mark.parametrize("kind", ["small", "wide", "sorted", "runs"])
def test_project_brute_force(kind):
    n = 4000
    v = rand_column(n, kind)
    sorted_pos = np.sort(RNG.choice(n, 900, replace=False)).astype(np.uint64) + np.uint64(77)
    unsorted_pos = RNG.integers(0, n, 700).astype(np.uint64) + np.uint64(77)
    for f, w, B in FMTS:
        d = O.encode(v, f, w, B)
        for pos in (sorted_pos, unsorted_pos):
            p = O.encode(pos, O.UNCOMPR)
            for of, ow, oB in [(O.FOR_BP, 0, 512), (O.UNCOMPR, 0, 0), (O.DYN_BP, 0, 128)]:
                got = O.decode(O.project(d, p, 77, of, ow, oB))
                assert np.array_equal(got, v[(pos - np.uint64(77)).astype(np.int64)])


def test_project_range_error():
    d = O.encode(np.arange(10, dtype=np.uint64), O.UNCOMPR)
    with pytest.raises(O.OracleError) as e:
        O.project(d, O.encode([3, 10], O.UNCOMPR))
    assert e.value.code == O.E_RANGE
    with pytest.raises(O.OracleError):
        O.project(d, O.encode([3], O.UNCOMPR), row_offset=5)


def py_sum(v):
    return int(sum(int(x) for x in v)) & M64


@pytest.mark.parametrize("kind", ["small", "wide", "sorted", "runs"])
def test_sum_brute_force_and_identities(kind):
    n = 3 * 512 + 11
    v = rand_column(n, kind)
    ref = py_sum(v)
    for f, w, B in FMTS:
        assert O.agg_sum(O.encode(v, f, w, B)) == ref
    # RLE identity: sum = sum value*length
    r = O.encode(v, O.RLE)
    assert sum(int(a) * int(l) for a, l in zip(r.payload[0::2], r.payload[1::2])) & M64 == ref
    # FOR identity: per block B*ref + sum codes; DELTA: B*base + sum (B-j)*d_j  (+ remainder)
    fo = O.encode(v, O.FOR_BP, 0, 512)
    de = O.encode(v, O.DELTA_BP, 0, 512)
    s_for, s_delta = 0, 0
    for b in range(fo.n_blocks):
        x = [int(t) for t in v[b * 512:(b + 1) * 512]]
        s_for += 512 * int(fo.ref[b]) + sum(t - int(fo.ref[b]) for t in x)
        d = [0] + [(x[j] - x[j - 1]) & M64 for j in range(1, 512)]
        s_delta += 512 * int(de.ref[b]) + sum((512 - j) * d[j] for j in range(512))
    tail = sum(int(t) for t in v[fo.n_blocks * 512:])
    assert (s_for + tail) & M64 == ref and (s_delta + tail) & M64 == ref


def test_sum_at_positions():
    v = rand_column(5000, "wide")
    pos = np.sort(RNG.choice(5000, 1000, replace=False)).astype(np.uint64)
    for f, w, B in FMTS:
        got = O.agg_sum(O.encode(v, f, w, B), O.encode(pos + np.uint64(3), O.DELTA_BP, 0, 512), 3)
        assert got == py_sum(v[pos.astype(np.int64)])


def test_grouped_sum_brute_force():
    n = 6000
    g = RNG.integers(0, 1000, n).astype(np.uint64)
    v = rand_column(n, "wide")
    expect = [0] * 1000
    for gi, vi in zip(g, v):
        expect[int(gi)] = (expect[int(gi)] + int(vi)) & M64
    for f, w, B in [(O.UNCOMPR, 0, 0), (O.STATIC_BP, 10, 0), (O.DYN_BP, 0, 512)]:
        got = O.agg_sum_grouped(O.encode(g, f, w, B), O.encode(v, O.DYN_BP, 0, 512), 1000)
        assert [int(x) for x in got] == expect
    with pytest.raises(O.OracleError):
        O.agg_sum_grouped(O.encode(g, O.UNCOMPR), O.encode(v, O.UNCOMPR), 999)


@pytest.mark.parametrize("kind", ["small", "sorted", "runs", "outlier"])
def test_morph_all_pairs(kind):
    v = rand_column(2048 * 2 + 100, kind)
    specs = [(O.UNCOMPR, 0, 0), (O.STATIC_BP, 64, 0), (O.DYN_BP, 0, 512), (O.FOR_BP, 0, 256),
             (O.DELTA_BP, 0, 2048), (O.RLE, 0, 0)]
    for a in specs:
        ca = O.encode(v, *a)
        for b in specs:
            m = O.morph(ca, *b)
            assert np.array_equal(O.decode(m), v)  # decode . morph = decode
            direct = O.encode(v, *b)  # direct morph == decompress-then-compress bytes
            for s in ("payload", "cw", "ref", "rem"):
                assert np.array_equal(getattr(m, s), getattr(direct, s))
        same = O.morph(ca, *a)  # identity morph is byte-identical
        for s in ("payload", "cw", "ref", "rem"):
            assert np.array_equal(getattr(same, s), getattr(ca, s))


@pytest.mark.parametrize("op", [O.EQ, O.NE, O.LT, O.LE, O.GT, O.GE, O.BETWEEN, O.IN_BITMAP])
def test_count_raw_brute_force(op):
    """orc_count_raw (the predicate count on a raw vector, D-11 / S:271)
    against numpy's own comparison operators, including the saturating
    constants 0 and 2^64-1 and an empty range."""
    v = np.concatenate([RNG.integers(0, 1 << 12, 3000, dtype=np.uint64),
                        np.array([0, 1, M64, M64 - 1, 4095, 4096], np.uint64)])
    bm = RNG.integers(0, 1 << 63, 70, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    cases = [(0, 0), (1, 4095), (2000, 2100), (M64, 0), (M64 - 1, M64), (2100, 2000)]
    for a, b in cases:
        bits = 4000 if op == O.IN_BITMAP else 0
        want = int(np_pred(v, op, a, b, bm, bits).sum())
        got = O.count_raw(v, op, a, b, bitmap=bm if op == O.IN_BITMAP else None, bitmap_bits=bits)
        assert got == want, (op, a, b)
