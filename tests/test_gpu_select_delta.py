"""GPU parity of select -> DELTA_BP{512} positions (the paper's positions
format) against the oracle, byte for byte, at sizes that span many
select tiles and output blocks with ragged tails: blocks straddling many empty
tiles, the final partial block, partial 512-row segments and block remainders,
every fast input layout (STATIC_BP at widths 1..64, UNCOMPR, DYN_BP / FOR_BP with
B >= 512, narrow and wide widths), the FOR code-domain predicate, bitmaps and
large row offsets (D-10)."""
import numpy as np
import pytest

import oracle as O
from tests.gpu_util import assert_same_image, get_ms, oracle_fmt, to_torch

pytestmark = pytest.mark.gpu

TILE = 32768


def run_both(v, fi, op, a, b=0, off=0, what=""):
    ms = get_ms()
    gi = ms.compress(to_torch(v), fi)
    oi = O.encode(v, *oracle_fmt(fi))
    g = ms.select(gi, op, a, b, row_offset=off, out_fmt=ms.delta_bp(512))
    o = O.select(oi, {ms.LT: O.LT, ms.EQ: O.EQ, ms.BETWEEN: O.BETWEEN, ms.GE: O.GE, ms.NE: O.NE}[op], a, b,
                 row_offset=off, out_fmt=O.DELTA_BP, out_block=512)
    assert_same_image(g, o, what)
    return g


@pytest.mark.parametrize("n", [1, 511, 512, 513, TILE - 1, TILE, TILE + 1, 3 * TILE + 12_345, 17 * TILE])
@pytest.mark.parametrize("sel", [1.0, 0.5, 0.0625, 0.004, 0.0])
def test_tiles_and_tails(n, sel):
    ms = get_ms()
    rng = np.random.default_rng(n + int(sel * 1000))
    v = rng.integers(0, 1 << 20, n).astype(np.uint64)
    thr = int(sel * (1 << 20))
    for fi in (ms.dyn_bp(512), ms.static_bp(20)):
        for off in (0, (1 << 40) + 3):
            run_both(v, fi, ms.LT, thr, off=off, what=f"n={n} sel={sel} {fi} off={off}")


def test_sparse_heads_span_many_tiles():
    """One match every ~3 tiles: every block's head comes from hundreds of
    predecessor tiles, most of them empty."""
    ms = get_ms()
    n = 1500 * TILE + 777
    v = np.ones(n, np.uint64)
    rng = np.random.default_rng(11)
    hit = rng.choice(n, 600, replace=False)
    v[hit] = 0
    v[n - 1] = 0  # a match in the last partial segment
    for fi in (ms.dyn_bp(512), ms.static_bp(1)):
        run_both(v, fi, ms.EQ, 0, off=123, what=f"sparse {fi}")


def test_clustered_runs_across_tiles():
    ms = get_ms()
    n = 40 * TILE + 999
    v = np.full(n, 9, np.uint64)
    rng = np.random.default_rng(3)
    for s in rng.integers(0, n - 70_000, 40):
        v[s:s + int(rng.integers(1, 70_000))] = 2
    run_both(v, ms.dyn_bp(512), ms.EQ, 2, what="clustered")


@pytest.mark.parametrize("w", [1, 2, 3, 7, 8, 15, 16, 17, 31, 32, 33, 40, 47, 63, 64])
def test_static_widths(w):
    ms = get_ms()
    rng = np.random.default_rng(w)
    n = 2 * TILE + 4097
    hi = (1 << w) if w < 64 else (1 << 64)
    v = rng.integers(0, hi, n, dtype=np.uint64, endpoint=False) if w < 64 else \
        rng.integers(0, 2**64 - 1, n, dtype=np.uint64, endpoint=True)
    thr = int(hi // 7) or 1
    run_both(v, ms.static_bp(w), ms.LT, thr, what=f"static w={w}")


def test_uncompressed_input():
    ms = get_ms()
    rng = np.random.default_rng(5)
    n = 3 * TILE + 100
    v = rng.integers(0, 2**64 - 1, n, dtype=np.uint64, endpoint=True)
    run_both(v, ms.uncompr(), ms.LT, 2**62, what="uncompr")
    run_both(v, ms.uncompr(), ms.GE, 2**63, off=7, what="uncompr GE")


@pytest.mark.parametrize("B", [512, 1024, 2048])
def test_block_formats_with_remainders(B):
    """DYN_BP / FOR_BP blocks of 512..2048 rows with a remainder of raw rows
    (decoded by random access at the end of the last tile), outliers that push
    some blocks past 32 bits (the wide kernel), and the FOR code-domain
    predicate."""
    ms = get_ms()
    rng = np.random.default_rng(B)
    n = 5 * TILE + B + 333
    v = rng.integers(0, 256, n).astype(np.uint64)
    out = rng.random(n) < 0.002
    v[out] = rng.integers(0, 1 << 40, int(out.sum())).astype(np.uint64)
    run_both(v, ms.dyn_bp(B), ms.EQ, 17, what=f"dyn{B} outliers")
    y = (10**6 + rng.integers(0, 1 << 20, n)).astype(np.uint64)
    run_both(y, ms.for_bp(B), ms.BETWEEN, 10**6 + 1000, 10**6 + 90_000, what=f"for{B}")
    run_both(y, ms.for_bp(B), ms.LT, 10**6 - 1, what=f"for{B} empty")


def test_bitmap_predicate_onepass():
    ms = get_ms()
    rng = np.random.default_rng(9)
    bits = 200_000
    words = rng.integers(0, 2**64 - 1, (bits + 63) // 64, dtype=np.uint64, endpoint=True)
    words &= rng.integers(0, 2**64 - 1, words.size, dtype=np.uint64, endpoint=True)
    n = 4 * TILE + 5
    v = rng.integers(0, 210_000, n).astype(np.uint64)
    X = ms.compress(to_torch(v), ms.static_bp(18))
    g = ms.select(X, ms.IN_BITMAP, bitmap=to_torch(words), bitmap_bits=bits, out_fmt=ms.delta_bp(512))
    o = O.select(O.encode(v, O.STATIC_BP, 18), O.IN_BITMAP, bitmap=words, bitmap_bits=bits,
                 out_fmt=O.DELTA_BP, out_block=512)
    assert_same_image(g, o, "bitmap")


def test_repeatable_and_single_sync():
    """The op is deterministic (same bytes on every call) and its result column
    owns a provable-capacity allocation (alloc_bytes >= footprint)."""
    ms = get_ms()
    rng = np.random.default_rng(1)
    n = 9 * TILE + 17
    v = rng.integers(0, 1 << 20, n).astype(np.uint64)
    X = ms.compress(to_torch(v), ms.dyn_bp(512))
    imgs = [ms.select(X, ms.LT, 1 << 16, out_fmt=ms.delta_bp(512)).images() for _ in range(3)]
    for im in imgs[1:]:
        for k in im:
            assert np.array_equal(im[k], imgs[0][k]), k
