"""GPU parity at every code width the compile-time-width kernels dispatch on,
byte-exact against the oracle:
- compress (cstream.cuh's word builder, one instantiation per width 1..64) into
  DYN_BP / FOR_BP / DELTA_BP at B = 512 and 2048, one block per width, each
  block's width forced exactly (its extreme value / spread / difference has the
  top bit set, D-4..D-7);
- the positions encoder (posdelta.cuh: pd_pack16<W> for W = 1..14 in the dense
  path, the listed blocks of the second launch for wider gaps), one 512-position
  block per width, its largest gap exactly 2^(w-1) (D-6: w = ebw(max d))."""
import numpy as np
import pytest

import oracle as O
from tests.gpu_util import assert_same_image, get_ms, to_torch

pytestmark = pytest.mark.gpu


def _blocks_every_width(kind, B, rng):
    out = []
    for w in range(1, 65):
        top = np.uint64(1) << np.uint64(w - 1)
        span = (top << np.uint64(1)) - np.uint64(1) if w < 64 else np.uint64(2**64 - 1)
        lo = rng.integers(0, 2**63, dtype=np.uint64)
        r = rng.integers(0, 2**63, B, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, B, dtype=np.uint64)
        r &= span
        if kind == "dyn":      # values < 2^w, one value with bit w-1 set
            v = r.copy()
            v[rng.integers(0, B)] |= top
        elif kind == "for":    # spread max - min = exactly a w-bit number with its top bit set
            v = r.copy()
            v[0] = 0
            v[rng.integers(1, B)] = span
            v = v + lo
        else:                  # delta: differences < 2^w, one with bit w-1 set (wrapping sums)
            d = r.copy()
            d[rng.integers(1, B)] |= top
            d[0] = lo
            v = np.cumsum(d, dtype=np.uint64)
        out.append(v.astype(np.uint64))
    return np.concatenate(out)


@pytest.mark.parametrize("B", [512, 2048])
@pytest.mark.parametrize("kind", ["dyn", "for", "delta"])
def test_compress_every_width(kind, B):
    ms = get_ms()
    rng = np.random.default_rng(1000 + B + len(kind))
    v = _blocks_every_width(kind, B, rng)
    v = np.concatenate([v, rng.integers(0, 2**40, 37, dtype=np.uint64)])  # a ragged remainder
    f = {"dyn": ms.dyn_bp(B), "for": ms.for_bp(B), "delta": ms.delta_bp(B)}[kind]
    of = {"dyn": O.DYN_BP, "for": O.FOR_BP, "delta": O.DELTA_BP}[kind]
    g = ms.compress(to_torch(v), f)
    o = O.encode(v, of, 0, B)
    assert_same_image(g, o, f"compress every width {kind} B={B}")
    assert np.array_equal(ms.to_u64_numpy(ms.decompress(g)), v)


def test_positions_every_width():
    """Block k of the selected rows has its largest gap 2^(w-1), w = 1..15 and two
    wider gaps (blocks whose mask span exceeds 512 words: the second launch)."""
    ms = get_ms()
    rng = np.random.default_rng(77)
    gaps = []
    for w in list(range(1, 16)) + [17, 20]:
        g = rng.integers(1, (1 << (w - 1)) + 1 if w > 1 else 2, 512).astype(np.int64)
        g[rng.integers(1, 512)] = 1 << (w - 1)
        gaps.append(g)
    gaps = np.concatenate(gaps + [np.ones(300, np.int64)])  # a partial last block
    pos = 5 + np.cumsum(gaps) - gaps[0]
    n = int(pos[-1]) + 1000
    x = np.ones(n, np.uint64)
    x[pos] = 0
    X = ms.compress(to_torch(x), ms.static_bp(1))
    oX = O.encode(x, O.STATIC_BP, 1)
    for off in (0, 1 << 36):
        g = ms.select(X, ms.EQ, 0, row_offset=off, out_fmt=ms.delta_bp(512))
        o = O.select(oX, O.EQ, 0, row_offset=off, out_fmt=O.DELTA_BP, out_block=512)
        assert_same_image(g, o, f"positions every width off={off}")
