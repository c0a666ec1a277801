"""GPU parity of select's positions encoder (mask -> DELTA_BP{B}, posdelta.cuh)
against the oracle, bit-exact, across the selectivities that switch between the
two walks of pos_slot (dense masks: rank-per-lane fast path; sparse masks: the
round-based walker), every block size it serves, block-boundary tails and large
row offsets; other positions formats through the slot and look-back encoders."""
import numpy as np
import pytest

import oracle as O
from tests.gpu_util import assert_same_image, get_ms, to_torch

pytestmark = pytest.mark.gpu

SELECTIVITY = [1.0, 0.9, 0.5, 0.125, 0.0625, 0.04, 0.031, 0.02, 0.0155, 0.005, 0.0003]


@pytest.mark.parametrize("sel", SELECTIVITY)
def test_positions_delta_bp(sel):
    ms = get_ms()
    rng = np.random.default_rng(int(sel * 1e6) + 7)
    for n in (600_001, 512 * 1024):
        v = rng.integers(0, 1 << 20, n).astype(np.uint64)
        thr = int(sel * (1 << 20))
        X = ms.compress(to_torch(v), ms.static_bp(20))
        oX = O.encode(v, O.STATIC_BP, 20)
        for B in (128, 256, 512):
            for off in (0, 1 << 40):
                g = ms.select(X, ms.LT, thr, row_offset=off, out_fmt=ms.delta_bp(B))
                o = O.select(oX, O.LT, thr, row_offset=off, out_fmt=O.DELTA_BP, out_block=B)
                assert_same_image(g, o, f"sel={sel} n={n} B={B} off={off}")


def test_positions_clustered():
    """Matches in dense clusters separated by long gaps: blocks mix both paths
    within one CTA tile."""
    ms = get_ms()
    rng = np.random.default_rng(5)
    n = 1 << 21
    v = np.full(n, 7, np.uint64)
    for s in rng.integers(0, n - 5000, 60):
        v[s:s + int(rng.integers(1, 5000))] = 1
    X = ms.compress(to_torch(v), ms.dyn_bp(512))
    oX = O.encode(v, O.DYN_BP, 0, 512)
    for B in (128, 512):
        g = ms.select(X, ms.EQ, 1, out_fmt=ms.delta_bp(B))
        o = O.select(oX, O.EQ, 1, out_fmt=O.DELTA_BP, out_block=B)
        assert_same_image(g, o, f"clustered B={B}")


@pytest.mark.parametrize("sel", [0.9, 0.0625, 0.003])
def test_positions_other_formats(sel):
    """Positions as UNCOMPR / STATIC_BP / DYN_BP / FOR_BP / RLE (slot encoder, and
    the deferred look-back encoder for RLE), byte-exact."""
    ms = get_ms()
    rng = np.random.default_rng(int(sel * 1000) + 3)
    n = 400_003
    v = rng.integers(0, 1 << 20, n).astype(np.uint64)
    thr = int(sel * (1 << 20))
    X = ms.compress(to_torch(v), ms.dyn_bp(512))
    oX = O.encode(v, O.DYN_BP, 0, 512)
    for fo, of in ((ms.uncompr(), (O.UNCOMPR, 0, 0)), (ms.static_bp(0), (O.STATIC_BP, 0, 0)),
                   (ms.static_bp(40), (O.STATIC_BP, 40, 0)), (ms.dyn_bp(512), (O.DYN_BP, 0, 512)),
                   (ms.for_bp(256), (O.FOR_BP, 0, 256)), (ms.dyn_bp(128), (O.DYN_BP, 0, 128)),
                   (ms.dyn_bp(2048), (O.DYN_BP, 0, 2048)), (ms.rle(), (O.RLE, 0, 0))):
        for off in (0, 1 << 33):
            g = ms.select(X, ms.LT, thr, row_offset=off, out_fmt=fo)
            o = O.select(oX, O.LT, thr, row_offset=off, out_fmt=of[0], out_width=of[1], out_block=of[2] or 512)
            assert_same_image(g, o, f"sel={sel} -> {fo} off={off}")
