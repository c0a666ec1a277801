"""CPU oracle, part 2 — TEST INFRASTRUCTURE ONLY (same rules as oracle/__init__.py:
only tests/, smoke() and bench.py's CPU legs may import it; the product never does).

Plain definitions of the operators beyond select / project / sum / morph that a
star-schema plan needs, and of the footprint-driven format choice, written on the
fully decoded columns (decode / encode are the C oracle's):

- format_sizes / choose_format: SPEC.md S:384-394 (estimate_size,
  select_format_footprint) and PAPER.md P:722-735 (cost-based selection, the
  compression-rate objective): the size of a format IS the footprint of the
  canonical image `encode_F(v)`; the choice is the minimum, ties broken by the
  fixed order UNCOMPR < STATIC_BP < DYN_BP < DELTA_BP < FOR_BP (simplest
  first), RLE last.
- intersect_sorted / merge_sorted: S:295-301 (sorted intersection / duplicate-free
  union of strictly increasing position lists; NotSorted -> E_INVALID).
- join_eq: S:302-306 (equi-join; all (i, j) with left[i] == right[j], ordered by
  probe-side scan order, then build-match order; build side = the smaller column,
  the right one on a tie).
- group: S:307-311 (dense group ids in first-occurrence order of the (previous id,
  key) combination; extents = first row of every group).
- calc_binary: S:318-321 (elementwise ADD / SUB / MUL mod 2^64).
Pins: tests/test_oracle_plan_ops.py.
"""
from __future__ import annotations

import numpy as np

import oracle as O

TIE_ORDER = (O.UNCOMPR, O.STATIC_BP, O.DYN_BP, O.DELTA_BP, O.FOR_BP, O.RLE)
ADD, SUB, MUL = 0, 1, 2
M64 = (1 << 64) - 1


def format_sizes(values, block_size: int = 512) -> list[int]:
    """Footprint of encode_F(values) for F in TIE_ORDER (STATIC_BP at its auto width)."""
    v = np.ascontiguousarray(values, np.uint64)
    out = []
    for f in TIE_ORDER:
        B = block_size if f in (O.DYN_BP, O.DELTA_BP, O.FOR_BP) else 0
        out.append(O.encode(v, f, 0, B).footprint())
    return out


def choose_format(values, block_size: int = 512) -> int:
    """The format of TIE_ORDER with the smallest footprint (first on a tie)."""
    s = format_sizes(values, block_size)
    return TIE_ORDER[min(range(len(s)), key=lambda i: (s[i], i))]


class NotSorted(ValueError):
    pass


def _strict(v):
    v = np.ascontiguousarray(v, np.uint64)
    if v.size > 1 and not np.all(v[1:] > v[:-1]):
        raise NotSorted("positions must be strictly increasing")
    return v


def intersect_sorted(a, b) -> np.ndarray:
    """Sorted intersection of two strictly increasing position lists."""
    a, b = _strict(a), _strict(b)
    return np.intersect1d(a, b, assume_unique=True).astype(np.uint64)


def merge_sorted(a, b) -> np.ndarray:
    """Sorted duplicate-free union of two strictly increasing position lists."""
    a, b = _strict(a), _strict(b)
    return np.union1d(a, b).astype(np.uint64)


def join_eq(left, right) -> tuple[np.ndarray, np.ndarray]:
    """(left positions, right positions) of all pairs with equal keys: the smaller
    column is the build side (the right one on a tie); pairs in probe-row order,
    then build-row order."""
    left = np.ascontiguousarray(left, np.uint64)
    right = np.ascontiguousarray(right, np.uint64)
    build_right = right.size <= left.size
    build, probe = (right, left) if build_right else (left, right)
    table: dict[int, list[int]] = {}
    for j, k in enumerate(build.tolist()):
        table.setdefault(k, []).append(j)
    pi, bj = [], []
    for i, k in enumerate(probe.tolist()):
        for j in table.get(k, ()):
            pi.append(i)
            bj.append(j)
    pi = np.array(pi, np.uint64)
    bj = np.array(bj, np.uint64)
    return (pi, bj) if build_right else (bj, pi)


def group(keys, prev_ids=None) -> tuple[np.ndarray, np.ndarray]:
    """(group ids, extents): id = rank of the (prev id, key) combination in order of
    first occurrence; extents[g] = row of the first occurrence of group g."""
    keys = np.ascontiguousarray(keys, np.uint64).tolist()
    prev = [0] * len(keys) if prev_ids is None else np.ascontiguousarray(prev_ids, np.uint64).tolist()
    if len(prev) != len(keys):
        raise ValueError("LengthMismatch")
    ids, ext, seen = [], [], {}
    for i, (p, k) in enumerate(zip(prev, keys)):
        g = seen.get((p, k))
        if g is None:
            g = seen[(p, k)] = len(ext)
            ext.append(i)
        ids.append(g)
    return np.array(ids, np.uint64), np.array(ext, np.uint64)


def calc_binary(op: int, a, b) -> np.ndarray:
    """Elementwise ADD / SUB / MUL mod 2^64 (Python integers, reduced mod 2^64)."""
    a = np.ascontiguousarray(a, np.uint64).tolist()
    b = np.ascontiguousarray(b, np.uint64).tolist()
    if len(a) != len(b):
        raise ValueError("LengthMismatch")
    f = {ADD: lambda x, y: x + y, SUB: lambda x, y: x - y, MUL: lambda x, y: x * y}[op]
    return np.array([f(x, y) & M64 for x, y in zip(a, b)], np.uint64)
