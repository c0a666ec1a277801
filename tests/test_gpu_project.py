"""GPU parity of project's encoders (positions.cuh ProjectSource gathers and the
streamed windows of projstream.cuh:
DELTA_BP{G} positions -> DYN_BP / FOR_BP data -> block output of size G or
UNCOMPR; G <= 512 through the slot encoder, larger G through the look-back
encoder) against the oracle, bit-exact: densities that do and do not fit the
32-block data window, data blocks wider than 32 bits, unsorted and repeated
positions, positions in the data remainder, a final partial positions block, and
the range error."""
import zlib

import numpy as np
import pytest

import oracle as O
from tests.gpu_util import assert_same_image, get_ms, oracle_fmt, to_torch

pytestmark = pytest.mark.gpu

@pytest.fixture(params=["slots", "lookback"])
def path(request):
    """Output block size 512 goes through the slot encoder (no look-back); 1024
    through the look-back encoder (warp_encode_kernel)."""
    return request.param


def _data(rng, n, kind):
    if kind == "narrow":
        return (np.uint64(10**6) + rng.integers(0, 1 << 20, n).astype(np.uint64))
    if kind == "mixed":  # some blocks wider than 32 bits
        v = rng.integers(0, 1 << 12, n).astype(np.uint64)
        hot = rng.random(n) < 0.002
        v[hot] = rng.integers(1 << 40, 1 << 63, int(hot.sum()), dtype=np.uint64)
        return v
    return rng.integers(0, 2**64 - 1, n, dtype=np.uint64, endpoint=True)  # wide


@pytest.mark.parametrize("kind", ["narrow", "mixed", "wide"])
@pytest.mark.parametrize("density", [0.5, 0.0625, 0.004])
def test_project_fast(kind, density, path):
    ms = get_ms()
    rng = np.random.default_rng(zlib.crc32(f"{kind}/{density}".encode()))
    n = 300_001
    off = 7_000_000_000
    v = _data(rng, n, kind)
    sel = np.nonzero(rng.random(n) < density)[0].astype(np.uint64) + np.uint64(off)
    for fd in (ms.for_bp(512), ms.dyn_bp(512), ms.for_bp(128), ms.dyn_bp(2048)):
        gd = ms.compress(to_torch(v), fd)
        od = O.encode(v, *oracle_fmt(fd))
        for G in ((512, 128) if path == "slots" else (1024, 2048)):
            fp = ms.delta_bp(G)
            gp = ms.compress(to_torch(sel), fp)
            op_ = O.encode(sel, *oracle_fmt(fp))
            outs = [ms.for_bp(G), ms.delta_bp(G), ms.dyn_bp(G)] + ([ms.uncompr()] if G == 512 else [])
            for fo in outs:
                gr = ms.project(gd, gp, off, fo)
                orr = O.project(od, op_, off, *oracle_fmt(fo))
                assert_same_image(gr, orr, f"project {kind} d={density} {fd} @ DELTA_BP{{{G}}} -> {fo}")


def test_project_fast_unsorted_and_repeated():
    ms = get_ms()
    rng = np.random.default_rng(11)
    n = 100_000
    v = _data(rng, n, "narrow")
    pos = np.sort(rng.integers(0, n, 20_000)).astype(np.uint64)   # repeated positions
    pos[1000:1600] = rng.integers(0, n, 600).astype(np.uint64)    # an unsorted stretch
    pos[-5:] = np.uint64(n - 1)                                     # the data remainder
    gd = ms.compress(to_torch(v), ms.for_bp(512))
    od = O.encode(v, O.FOR_BP, 0, 512)
    gp = ms.compress(to_torch(pos), ms.delta_bp(512))
    op_ = O.encode(pos, O.DELTA_BP, 0, 512)
    for fo in (ms.for_bp(512), ms.uncompr(), ms.delta_bp(512)):
        assert_same_image(ms.project(gd, gp, 0, fo), O.project(od, op_, 0, *oracle_fmt(fo)), f"-> {fo}")


def test_project_fast_range_error():
    ms = get_ms()
    v = np.arange(5000, dtype=np.uint64)
    gd = ms.compress(to_torch(v), ms.for_bp(512))
    pos = np.arange(0, 1024, dtype=np.uint64) * 4
    pos[700] = 5000  # one past the end
    gp = ms.compress(to_torch(np.sort(pos)), ms.delta_bp(512))
    with pytest.raises(ms.MsError) as e:
        ms.project(gd, gp, 0, ms.for_bp(512))
    assert e.value.code == 4  # MS_E_RANGE


def _ran(ms, fn):
    ms.profile_read()
    ms.profile_enable(True)
    try:
        out = fn()
        return out, set(ms.profile_read())
    finally:
        ms.profile_enable(False)


@pytest.mark.parametrize("kind", ["narrow", "w40", "zeros"])
@pytest.mark.parametrize("fd_name", ["for128", "for512", "dyn128", "dyn2048"])
def test_project_stream(kind, fd_name):
    """Dense DELTA_BP{512} positions stream the data windows through shared memory
    (projstream.cuh); the output equals the oracle's and the gather path's
    (MS_FLAG_GATHER) byte for byte. The positions mix dense stretches (streamed
    windows), a sparse stretch (windows above the stage cap: gather fallback), rows
    in the data remainder, a final partial block, and a row offset."""
    ms = get_ms()
    rng = np.random.default_rng(zlib.crc32(f"stream/{kind}/{fd_name}".encode()))
    n = 2_000_000 + 333
    off = 5_000_000_000
    if kind == "w40":  # codes wider than 32 bits
        v = rng.integers(0, 1 << 40, n).astype(np.uint64)
    else:
        v = _data(rng, n, "narrow")
    if kind == "zeros":
        v[: n // 2] = 0  # zero-width data blocks: windows of zero payload bytes
    keep = rng.random(n) < (1 / 4 if kind == "w40" else 1 / 8)
    keep[700_000:1_100_000] = rng.random(400_000) < 1 / 900    # sparse stretch
    keep[n - 200:] = True                                          # the data remainder
    sel = np.nonzero(keep)[0].astype(np.uint64) + np.uint64(off)
    fd = {"for128": ms.for_bp(128), "for512": ms.for_bp(512), "dyn128": ms.dyn_bp(128),
          "dyn2048": ms.dyn_bp(2048)}[fd_name]
    gd = ms.compress(to_torch(v), fd)
    od = O.encode(v, *oracle_fmt(fd))
    gp = ms.compress(to_torch(sel), ms.delta_bp(512))
    op_ = O.encode(sel, O.DELTA_BP, 0, 512)
    assert gp.n % 512 != 0
    for fo in (ms.for_bp(512), ms.dyn_bp(512), ms.delta_bp(512)):
        gr, names = _ran(ms, lambda: ms.project(gd, gp, off, fo))
        assert "project_stream" in names, names
        orr = O.project(od, op_, off, *oracle_fmt(fo))
        assert_same_image(gr, orr, f"stream {kind} {fd} -> {fo}")
        gg, names_g = _ran(ms, lambda: ms.project(gd, gp, off, fo, flags=ms.FLAG_GATHER))
        assert "project_stream" not in names_g and "project_slot" in names_g
        assert_same_image(gg, orr, f"gather {kind} {fd} -> {fo}")


def test_project_stream_unsorted_and_range():
    """Positions outside their block's window (an unsorted stretch, repeats across
    block boundaries) are read directly; one past the end is MS_E_RANGE."""
    ms = get_ms()
    rng = np.random.default_rng(5)
    n = 400_000
    v = _data(rng, n, "narrow")
    pos = np.sort(rng.integers(0, n, 60_000)).astype(np.uint64)
    pos[20_000:20_700] = rng.integers(0, n, 700).astype(np.uint64)
    gd = ms.compress(to_torch(v), ms.for_bp(512))
    od = O.encode(v, O.FOR_BP, 0, 512)
    gp = ms.compress(to_torch(pos), ms.delta_bp(512))
    op_ = O.encode(pos, O.DELTA_BP, 0, 512)
    gr, names = _ran(ms, lambda: ms.project(gd, gp, 0, ms.for_bp(512)))
    assert "project_stream" in names
    assert_same_image(gr, O.project(od, op_, 0, O.FOR_BP, 0, 512), "unsorted")
    bad = np.sort(rng.integers(0, n, 60_000)).astype(np.uint64)
    bad[30_000] = n  # one past the end, inside a dense stretch
    bad = np.sort(bad)
    with pytest.raises(ms.MsError) as e:
        ms.project(gd, ms.compress(to_torch(bad), ms.delta_bp(512)), 0, ms.for_bp(512))
    assert e.value.code == 4  # MS_E_RANGE


def test_project_stream_stage_reuse():
    """More output blocks per CTA than stages (7 stages x 148 CTAs): every stage
    and consumer pair is reused many times; byte-exact against the oracle."""
    ms = get_ms()
    rng = np.random.default_rng(77)
    n = 8_000_000 + 4321
    v = _data(rng, n, "narrow")
    sel = np.nonzero(rng.random(n) < 1 / 8)[0].astype(np.uint64)
    gd = ms.compress(to_torch(v), ms.for_bp(512))
    gp = ms.compress(to_torch(sel), ms.delta_bp(512))
    assert gp.n // 512 > 7 * 148  # > 7 blocks per CTA
    gr, names = _ran(ms, lambda: ms.project(gd, gp, 0, ms.for_bp(512)))
    assert "project_stream" in names
    assert_same_image(gr, O.project(O.encode(v, O.FOR_BP, 0, 512), O.encode(sel, O.DELTA_BP, 0, 512), 0,
                                    O.FOR_BP, 0, 512), "stage reuse")
