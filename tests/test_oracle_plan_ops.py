"""Pins of oracle/plan_ops.py (PAPER.md P:577-582,
722-735): SPEC's worked examples, the paper's best formats per column of Table
tab:datach on the size objective, brute force (nested loops / set semantics) on
small random inputs, and algebraic identities."""
import itertools

import numpy as np
import pytest

import oracle as O
import synth
from oracle import plan_ops as P

RNG = np.random.default_rng(17)


@pytest.mark.parametrize("col,best", [("C1.plain", O.STATIC_BP), ("C2.plain", O.DYN_BP), ("C3.Y", O.FOR_BP),
                                      ("C4.Y", O.DELTA_BP)])
def test_choose_format_paper_columns(col, best):
    """C1 -> static BP, C2 -> SIMD-BP512 (DYN_BP), C3 -> FOR, C4 -> DELTA
    (the paper's best input formats; on the footprint objective as S:394 asserts)."""
    v = synth.gen_host(col, 1 << 16)
    assert P.choose_format(v, 512) == best


def test_format_sizes_closed_forms():
    """Footprints against the size laws of SURVEY.md §8(c) c.2 computed by hand."""
    n = 3 * 512 + 100
    v = RNG.integers(0, 1 << 13, n).astype(np.uint64)
    s = dict(zip(P.TIE_ORDER, P.format_sizes(v, 512)))
    w = int(v.max()).bit_length()
    assert s[O.UNCOMPR] == 8 * n
    assert s[O.STATIC_BP] == 8 * ((n * w + 63) // 64)
    blocks = v[:3 * 512].reshape(3, 512)
    dyn = sum(512 * int(b.max()).bit_length() // 8 for b in blocks)
    assert s[O.DYN_BP] == dyn + 4 * 4 + 8 * 100
    fr = sum(512 * int(b.max() - b.min()).bit_length() // 8 for b in blocks)
    assert s[O.FOR_BP] == fr + 4 * 4 + 8 * 3 + 8 * 100
    dl = sum(512 * max(int((int(x) - int(y)) % (1 << 64)).bit_length() for x, y in zip(b[1:], b[:-1])) // 8
             for b in blocks)
    assert s[O.DELTA_BP] == dl + 4 * 4 + 8 * 3 + 8 * 100
    assert s[O.RLE] == 16 * (1 + int(np.count_nonzero(v[1:] != v[:-1])))


def test_choose_format_ties():
    """Constant column: zero-payload formats tie; the fixed order decides;
    RLE (one run) is smallest of all."""
    v = np.full(5000, 7, np.uint64)
    s = P.format_sizes(v, 512)
    assert s[P.TIE_ORDER.index(O.DELTA_BP)] == s[P.TIE_ORDER.index(O.FOR_BP)]
    assert P.choose_format(v, 512) == O.RLE
    z = np.zeros(4096, np.uint64)  # DYN_BP at width 0 has the smallest block image
    assert P.choose_format(z[:4095], 512) in (O.RLE,)


def test_intersect_merge_examples_and_sets():
    assert P.intersect_sorted([1, 3, 5], [3, 5, 7]).tolist() == [3, 5]
    assert P.merge_sorted([1, 3], [2, 3]).tolist() == [1, 2, 3]
    for _ in range(20):
        a = np.unique(RNG.integers(0, 300, RNG.integers(0, 80)))
        b = np.unique(RNG.integers(0, 300, RNG.integers(0, 80)))
        assert P.intersect_sorted(a, b).tolist() == sorted(set(a.tolist()) & set(b.tolist()))
        assert P.merge_sorted(a, b).tolist() == sorted(set(a.tolist()) | set(b.tolist()))
        assert P.intersect_sorted(a, a).tolist() == a.tolist()
        assert P.merge_sorted(a, []).tolist() == a.tolist()
    with pytest.raises(P.NotSorted):
        P.intersect_sorted([3, 1], [1])


def test_join_eq_example_and_nested_loops():
    lp, rp = P.join_eq([1, 2, 3], [2, 2, 4])
    assert lp.tolist() == [1, 1] and rp.tolist() == [0, 1]
    lp, rp = P.join_eq([1, 2], [5, 6, 7])
    assert lp.size == 0 and rp.size == 0
    for _ in range(20):
        L = RNG.integers(0, 12, RNG.integers(1, 40)).astype(np.uint64)
        R = RNG.integers(0, 12, RNG.integers(1, 40)).astype(np.uint64)
        lp, rp = P.join_eq(L, R)
        pairs = [(i, j) for i, j in itertools.product(range(L.size), range(R.size)) if L[i] == R[j]]
        assert sorted(zip(lp.tolist(), rp.tolist())) == sorted(pairs)
        # probe order, then build order: the probe side's positions are non-decreasing
        probe = lp if R.size <= L.size else rp
        assert np.all(probe[1:] >= probe[:-1])


def test_group_examples_and_dictionary():
    ids, ext = P.group([7, 8, 7])
    assert ids.tolist() == [0, 1, 0] and ext.tolist() == [0, 1]
    ids, ext = P.group([5, 6, 5], [0, 0, 1])
    assert ids.tolist() == [0, 1, 2] and ext.tolist() == [0, 1, 2]
    for _ in range(10):
        k = RNG.integers(0, 9, 200).astype(np.uint64)
        ids, ext = P.group(k)
        assert np.array_equal(k[ext], np.array(list(dict.fromkeys(k.tolist())), np.uint64))
        assert np.array_equal(k[ext][ids], k)  # every row maps to a group of its own key
        assert np.all(np.diff(ext.astype(np.int64)) > 0)  # first-occurrence order


def test_calc_binary():
    assert P.calc_binary(P.MUL, [2, 3], [4, 5]).tolist() == [8, 15]
    x = RNG.integers(0, 2**64 - 1, 100, dtype=np.uint64, endpoint=True)
    assert np.array_equal(P.calc_binary(P.ADD, x, np.zeros(100, np.uint64)), x)
    assert np.array_equal(P.calc_binary(P.SUB, x, x), np.zeros(100, np.uint64))
    big = np.array([2**63], np.uint64)
    assert P.calc_binary(P.ADD, big, big).tolist() == [0]
    assert P.calc_binary(P.MUL, big, np.array([2], np.uint64)).tolist() == [0]
