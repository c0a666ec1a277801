"""BASELINE.json configs c1..c5 end to end on the GPU, through the C ABI.

Reduced sizes: every intermediate image (positions, projected columns, morph
outputs) is compared byte for byte with the oracle's on the same seeded rows.
Full sizes: the chain runs at the config's own size and its counts, sums and
grouped sums must equal tests/golden/config_anchors.json (written by
tools/make_anchors.py from oracle/ only); sampled row ranges of the full-size
positions are additionally checked against the oracle's select on those rows.
"""
import json
import os

import numpy as np
import pytest

import oracle as O
import synth
from tests.gpu_util import assert_same_image, get_ms, oracle_fmt, to_torch

pytestmark = pytest.mark.gpu

ANCHORS = os.path.join(os.path.dirname(__file__), "golden", "config_anchors.json")


def anchors():
    if not os.path.exists(ANCHORS):
        pytest.skip("tests/golden/config_anchors.json missing (python tools/make_anchors.py)")
    return json.load(open(ANCHORS))


def dev(name, n, start=0):
    return synth.gen_torch(name, n, start=start)


def check_sampled_positions(ms, pos, X_oracle_fn, op, a, b=0, samples=((0, 1 << 16),)):
    """Positions inside each sampled row range [lo, hi) must equal the oracle's
    select over exactly those rows (offset to global row ids)."""
    p = ms.to_u64_numpy(ms.decompress(pos))
    for lo, hi in samples:
        ox = O.encode(X_oracle_fn(hi - lo, lo), O.UNCOMPR)
        want = O.decode(O.select(ox, op, a, b, row_offset=lo, out_fmt=O.UNCOMPR))
        got = p[(p >= lo) & (p < hi)]
        assert np.array_equal(got, want), (lo, hi, got[:5], want[:5])


# ------------------------------------------------------------------ c1
def test_c1_full():
    ms = get_ms()
    n = 1 << 20
    X = ms.compress(dev("c1.X", n), ms.static_bp(10))
    pos = ms.select(X, ms.LT, 102, out_fmt=ms.delta_bp(512))
    xp = ms.project(X, pos, 0, ms.for_bp(512))
    ox = O.encode(synth.gen_host("c1.X", n), O.STATIC_BP, 10)
    opos = O.select(ox, O.LT, 102, out_fmt=O.DELTA_BP, out_block=512)
    assert_same_image(X, ox, "c1 X")
    assert_same_image(pos, opos, "c1 positions")
    assert_same_image(xp, O.project(ox, opos, 0, O.FOR_BP, 0, 512), "c1 X[pos]")
    s = ms.u64(ms.agg_sum(xp))
    assert s == ms.u64(ms.agg_sum(X, pos)) == O.agg_sum(ox, opos)


# ------------------------------------------------------------------ c2
def c2_chain(ms, n, start=0):
    X = ms.compress(dev("c2.X", n, start), ms.dyn_bp(512))
    Y = ms.compress(dev("c2.Y", n, start), ms.for_bp(512))
    pos = ms.select(X, ms.EQ, 17, row_offset=start, out_fmt=ms.delta_bp(512))
    yp = ms.project(Y, pos, start, ms.for_bp(512))
    yu = ms.project(Y, pos, start, ms.uncompr())
    return X, Y, pos, yp, yu


def test_c2_reduced():
    ms = get_ms()
    n = 1 << 22
    X, Y, pos, yp, yu = c2_chain(ms, n)
    ox = O.encode(synth.gen_host("c2.X", n), O.DYN_BP, 0, 512)
    oy = O.encode(synth.gen_host("c2.Y", n), O.FOR_BP, 0, 512)
    opos = O.select(ox, O.EQ, 17, out_fmt=O.DELTA_BP, out_block=512)
    assert_same_image(X, ox, "c2 X")
    assert_same_image(Y, oy, "c2 Y")
    assert_same_image(pos, opos, "c2 positions")
    assert_same_image(yp, O.project(oy, opos, 0, O.FOR_BP, 0, 512), "c2 Y' FOR")
    assert_same_image(yu, O.project(oy, opos, 0, O.UNCOMPR), "c2 Y' UNCOMPR")
    assert ms.u64(ms.agg_sum(yp)) == ms.u64(ms.agg_sum(yu)) == ms.u64(ms.agg_sum(Y, pos))


def test_c2_full():
    ms = get_ms()
    a = anchors()["c2"]
    X, Y, pos, yp, yu = c2_chain(ms, a["n"])
    assert pos.n == a["count"]
    assert ms.u64(ms.agg_sum(yp)) == ms.u64(ms.agg_sum(yu)) == a["sum_projected"]
    # full-size image anchors (oracle-computed: 1,476,652 / 2,624,044 B)
    assert pos.footprint() == a["positions_bytes"]
    assert yp.footprint() == a["yp_for_bytes"]
    assert yu.footprint() == a["yp_uncompr_bytes"]
    check_sampled_positions(ms, pos, lambda m, s: synth.gen_host("c2.X", m, s), O.EQ, 17,
                            samples=((0, 1 << 20), (a["n"] - (1 << 20), a["n"])))


# ------------------------------------------------------------------ c3
def c3_chain(ms, x, lo, hi):
    t = to_torch(x)
    R = ms.compress(t, ms.rle())
    D = ms.compress(t, ms.delta_bp(2048))
    pr = ms.select(R, ms.BETWEEN, lo, hi, out_fmt=ms.delta_bp(512))
    pd = ms.select(D, ms.BETWEEN, lo, hi, out_fmt=ms.delta_bp(512))
    m1 = ms.morph(R, ms.delta_bp(2048))
    m2 = ms.morph(D, ms.static_bp(0))
    return R, D, pr, pd, m1, m2


def test_c3_reduced():
    ms = get_ms()
    n = 1 << 22
    x = synth.gen_host("c3.x", n)
    lo, hi = int(x[n // 4]), int(x[n // 2])  # the config's range scaled to this prefix
    R, D, pr, pd, m1, m2 = c3_chain(ms, x, lo, hi)
    oR = O.encode(x, O.RLE)
    oD = O.encode(x, O.DELTA_BP, 0, 2048)
    opos = O.select(oD, O.BETWEEN, lo, hi, out_fmt=O.DELTA_BP, out_block=512)
    assert_same_image(R, oR, "c3 RLE")
    assert_same_image(D, oD, "c3 DELTA_BP{2048}")
    assert_same_image(pr, opos, "c3 positions from RLE")
    assert_same_image(pd, opos, "c3 positions from DELTA_BP")
    assert_same_image(m1, oD, "c3 morph RLE -> DELTA_BP{2048}")
    assert_same_image(m2, O.morph(oD, O.STATIC_BP, 0, 0), "c3 morph DELTA_BP -> STATIC_BP")
    s = O.agg_sum(oD, opos)
    assert ms.u64(ms.agg_sum(R, pr)) == ms.u64(ms.agg_sum(D, pd)) == s


def test_c3_full():
    ms = get_ms()
    a = anchors()["c3"]
    x_dev = dev("c3.x", a["n"])
    R = ms.compress(x_dev, ms.rle())
    D = ms.compress(x_dev, ms.delta_bp(2048))
    del x_dev
    assert R.n_runs == a["rle_runs"]
    assert 8 * D.payload_words == a["delta_bp2048_payload_bytes"]
    pr = ms.select(R, ms.BETWEEN, 10**6, 2 * 10**6, out_fmt=ms.delta_bp(512))
    pd = ms.select(D, ms.BETWEEN, 10**6, 2 * 10**6, out_fmt=ms.delta_bp(512))
    assert pr.n == pd.n == a["count"]
    assert pd.footprint() == a["positions_bytes"]
    assert_same_image(pr, O.encode(ms.to_u64_numpy(ms.decompress(pd)), O.DELTA_BP, 0, 512), "c3 pos RLE vs DELTA")
    p = ms.to_u64_numpy(ms.decompress(pd))
    assert int(p[0]) == a["first"] and int(p[-1]) == a["last"]
    assert ms.u64(ms.agg_sum(R, pr)) == ms.u64(ms.agg_sum(D, pd)) == a["sum_selected"]
    m1 = ms.morph(R, ms.delta_bp(2048))
    check_sampled_delta_blocks(m1, a["n"], 2048, "c3 morph RLE -> DELTA_BP{2048}")
    assert 8 * m1.payload_words == a["delta_bp2048_payload_bytes"]
    m2 = ms.morph(D, ms.static_bp(0))
    assert m2.fmt.bit_width == a["static_bp_auto_width"]
    check_sampled_static_rows(m2, a["n"], "c3 morph DELTA_BP{2048} -> STATIC_BP{auto}")
    assert ms.u64(ms.agg_sum(m2)) == ms.u64(ms.agg_sum(D)) == a["sum_all"]


SAMPLE_BLOCKS = (0, 1, 777, 65_536, 131_071, 200_003, 262_143)


def check_sampled_delta_blocks(col, n, B, what):
    """Full-size DELTA_BP column vs the oracle, block by block: blocks are
    independent (D-6), so block b's payload words, cw step and base equal the
    oracle's image of rows [bB, bB + B) alone (c3 rows from the host generator)."""
    img = col.images()
    for b in SAMPLE_BLOCKS:
        if b >= n // B:
            continue
        oc = O.encode(synth.gen_host("c3.x", B, b * B), O.DELTA_BP, 0, B)
        w0, w1 = int(img["cw"][b]), int(img["cw"][b + 1])
        assert w1 - w0 == int(oc.cw[1]), (what, b)
        assert int(img["ref"][b]) == int(oc.ref[0]), (what, b)
        got = img["payload"][w0 * (B // 64):w1 * (B // 64)]
        assert np.array_equal(got, oc.payload), (what, b)


def check_sampled_static_rows(col, n, what):
    """Full-size STATIC_BP{w} column vs the oracle on sampled 64-row groups: rows
    [r0, r0 + 64) with 64 | r0 occupy exactly words [r0 w / 64, (r0 + 64) w / 64)."""
    w = col.fmt.bit_width
    pay = col.images()["payload"]
    for b in SAMPLE_BLOCKS:
        r0 = (b * 2048 + 64 * (b % 29)) % (n - 64)
        r0 -= r0 % 64
        oc = O.encode(synth.gen_host("c3.x", 64, r0), O.STATIC_BP, w)
        got = pay[r0 * w // 64:(r0 + 64) * w // 64]
        assert np.array_equal(got, oc.payload), (what, r0)


# ------------------------------------------------------------------ c4 (D-16 chain)
def c4_chain(ms, n, start=0):
    D = synth.D4
    bm = to_torch(synth.bitmap_c4())
    gattr = ms.compress(dev("c4.gattr", D[3]), ms.static_bp(10))
    k0 = ms.compress(dev("c4.k0", n, start), ms.static_bp(12))
    k1 = ms.compress(dev("c4.k1", n, start), ms.static_bp(18))
    k3 = ms.compress(dev("c4.k3", n, start), ms.static_bp(17))
    m1 = ms.compress(dev("c4.m1", n, start), ms.dyn_bp(512))
    m2 = ms.compress(dev("c4.m2", n, start), ms.dyn_bp(512))
    pos1 = ms.select(k0, ms.BETWEEN, 0, 365, row_offset=start, out_fmt=ms.delta_bp(512))
    k1p = ms.project(k1, pos1, start, ms.static_bp(18))
    idx = ms.select(k1p, ms.IN_BITMAP, bitmap=bm, bitmap_bits=D[1], out_fmt=ms.delta_bp(512))
    pos2 = ms.project(pos1, idx, 0, ms.delta_bp(512))
    m1p = ms.project(m1, pos2, start, ms.dyn_bp(512))
    m2p = ms.project(m2, pos2, start, ms.dyn_bp(512))
    k3p = ms.project(k3, pos2, start, ms.static_bp(17))
    gid = ms.project(gattr, k3p, 0, ms.static_bp(10))
    g1 = ms.to_u64_numpy(ms.agg_sum_grouped(gid, m1p, 1000))
    g2 = ms.to_u64_numpy(ms.agg_sum_grouped(gid, m2p, 1000))
    return dict(pos1=pos1, k1p=k1p, idx=idx, pos2=pos2, m1p=m1p, m2p=m2p, k3p=k3p, gid=gid, g1=g1, g2=g2)


def test_c4_reduced():
    ms = get_ms()
    n = 1 << 22
    D = synth.D4
    g = c4_chain(ms, n)
    bm = synth.bitmap_c4()
    gattr = O.encode(synth.gen_host("c4.gattr", D[3]), O.STATIC_BP, 10)
    k0 = O.encode(synth.gen_host("c4.k0", n), O.STATIC_BP, 12)
    k1 = O.encode(synth.gen_host("c4.k1", n), O.STATIC_BP, 18)
    k3 = O.encode(synth.gen_host("c4.k3", n), O.STATIC_BP, 17)
    m1 = O.encode(synth.gen_host("c4.m1", n), O.DYN_BP, 0, 512)
    m2 = O.encode(synth.gen_host("c4.m2", n), O.DYN_BP, 0, 512)
    pos1 = O.select(k0, O.BETWEEN, 0, 365, out_fmt=O.DELTA_BP, out_block=512)
    k1p = O.project(k1, pos1, 0, O.STATIC_BP, 18, 0)
    idx = O.select(k1p, O.IN_BITMAP, bitmap=bm, bitmap_bits=D[1], out_fmt=O.DELTA_BP, out_block=512)
    pos2 = O.project(pos1, idx, 0, O.DELTA_BP, 0, 512)
    m1p = O.project(m1, pos2, 0, O.DYN_BP, 0, 512)
    m2p = O.project(m2, pos2, 0, O.DYN_BP, 0, 512)
    k3p = O.project(k3, pos2, 0, O.STATIC_BP, 17, 0)
    gid = O.project(gattr, k3p, 0, O.STATIC_BP, 10, 0)
    for name, oc in (("pos1", pos1), ("k1p", k1p), ("idx", idx), ("pos2", pos2), ("m1p", m1p), ("m2p", m2p),
                     ("k3p", k3p), ("gid", gid)):
        assert_same_image(g[name], oc, f"c4 {name}")
    assert np.array_equal(g["g1"], O.agg_sum_grouped(gid, m1p, 1000))
    assert np.array_equal(g["g2"], O.agg_sum_grouped(gid, m2p, 1000))


def test_c4_formats_chosen_at_run_time():
    """BJ.c4 with every intermediate re-encoded in the format the GPU's exact-size
    profile chooses (ms_format_sizes: the compression-rate objective of P:722-735,
    ties by S:392's order): each choice equals the oracle's choice on the same
    values, and the chain's grouped sums are unchanged (format transparency)."""
    ms = get_ms()
    n = 1 << 22
    from oracle import plan_ops as P
    g = c4_chain(ms, n)
    chosen = {}
    for name in ("pos1", "k1p", "idx", "pos2", "m1p", "m2p", "k3p", "gid"):
        c = g[name]
        sizes, best = ms.format_sizes(c, 512)
        vals = ms.to_u64_numpy(ms.decompress(c))
        assert best.format == P.choose_format(vals, 512), name
        assert [sizes[k] for k in ms.CANDIDATES] == P.format_sizes(vals, 512), name
        m = ms.morph(c, best)
        assert m.footprint() == min(sizes.values()), name
        assert np.array_equal(ms.to_u64_numpy(ms.decompress(m)), vals), name
        chosen[name] = (best, m)
    # the grouped sums from the re-encoded intermediates equal the fixed-format chain's
    g1 = ms.to_u64_numpy(ms.agg_sum_grouped(chosen["gid"][1], chosen["m1p"][1], 1000))
    g2 = ms.to_u64_numpy(ms.agg_sum_grouped(chosen["gid"][1], chosen["m2p"][1], 1000))
    assert np.array_equal(g1, g["g1"]) and np.array_equal(g2, g["g2"])


def test_c4_full():
    ms = get_ms()
    a = anchors()["c4"]
    g = c4_chain(ms, a["n"])
    assert g["pos1"].n == a["count_pos1"]
    assert g["pos2"].n == a["count_pos2"]
    # full-size image anchors (oracle-computed; 66,462,044 / 4,719,624 B)
    assert g["pos1"].footprint() == a["pos1_bytes"]
    assert g["pos2"].footprint() == a["pos2_bytes"]
    assert ms.u64(ms.agg_sum(g["m1p"])) == a["sum_m1"]
    assert ms.u64(ms.agg_sum(g["m2p"])) == a["sum_m2"]
    assert [int(x) for x in g["g1"]] == a["grouped_m1"]
    assert [int(x) for x in g["g2"]] == a["grouped_m2"]


# ------------------------------------------------------------------ c5 (sharded by row range)
def test_c5_two_shards_reduced():
    """Two row-range shards on one GPU (the multi-GPU layout, D-18): per-shard
    images equal the oracle's over the shard's rows, global row ids, and the
    shard sums add up to the single-column sum."""
    ms = get_ms()
    from paper_2004_09350_b200 import dist as D
    n = 1 << 22
    total = 0
    for s in range(2):
        start, end = D.shard_range(n, 2, s)
        m = end - start
        X = ms.compress(dev("c5.X", m, start), ms.dyn_bp(512))
        Y = ms.compress(dev("c5.Y", m, start), ms.for_bp(512))
        pos = ms.select(X, ms.LT, 1 << 16, row_offset=start, out_fmt=ms.delta_bp(512))
        yp = ms.project(Y, pos, start, ms.for_bp(512))
        ox = O.encode(synth.gen_host("c5.X", m, start), O.DYN_BP, 0, 512)
        oy = O.encode(synth.gen_host("c5.Y", m, start), O.FOR_BP, 0, 512)
        opos = O.select(ox, O.LT, 1 << 16, row_offset=start, out_fmt=O.DELTA_BP, out_block=512)
        assert_same_image(pos, opos, f"c5 shard {s} positions")
        assert_same_image(yp, O.project(oy, opos, start, O.FOR_BP, 0, 512), f"c5 shard {s} Y'")
        total += ms.u64(ms.agg_sum(yp))
    ox = O.encode(synth.gen_host("c5.X", n), O.DYN_BP, 0, 512)
    oy = O.encode(synth.gen_host("c5.Y", n), O.FOR_BP, 0, 512)
    opos = O.select(ox, O.LT, 1 << 16, out_fmt=O.DELTA_BP, out_block=512)
    assert total % (1 << 64) == O.agg_sum(oy, opos)


def test_c5_full():
    ms = get_ms()
    a = anchors()["c5"]
    n = a["n"]
    X = ms.compress(dev("c5.X", n), ms.dyn_bp(512))
    Y = ms.compress(dev("c5.Y", n), ms.for_bp(512))
    pos = ms.select(X, ms.LT, 1 << 16, out_fmt=ms.delta_bp(512))
    assert pos.n == a["count"]
    yp = ms.project(Y, pos, 0, ms.for_bp(512))
    assert ms.u64(ms.agg_sum(yp)) == a["sum_projected"]
    # full-size image anchors (oracle-computed; 245,585,644 / 677,386,156 B)
    assert pos.footprint() == a["positions_bytes"]
    assert yp.footprint() == a["yp_bytes"]
    del Y, yp
    check_sampled_positions(ms, pos, lambda m, s: synth.gen_host("c5.X", m, s), O.LT, 1 << 16,
                            samples=((0, 1 << 20), (n // 2, n // 2 + (1 << 20)), (n - (1 << 20), n)))


def test_c5_eight_shards_full():
    """BJ.c5's G = 8 layout emulated on one GPU, shard after shard (D-18, SURVEY.md
    §8(e)): each 2^29-row shard's count equals the oracle's per-shard count, each
    shard's positions / Y' image sizes equal the oracle's images of that shard,
    the C1 offsets are the exclusive scan of the counts, and the shard sums add
    up (mod 2^64) to the single-column sum."""
    ms = get_ms()
    from paper_2004_09350_b200 import dist as D
    a = anchors()["c5"]
    n, G = a["n"], 8
    counts, total = [], 0
    for s in range(G):
        start, end = D.shard_range(n, G, s)
        m = end - start
        X = ms.compress(dev("c5.X", m, start), ms.dyn_bp(512))
        Y = ms.compress(dev("c5.Y", m, start), ms.for_bp(512))
        pos = ms.select(X, ms.LT, 1 << 16, row_offset=start, out_fmt=ms.delta_bp(512))
        yp = ms.project(Y, pos, start, ms.for_bp(512))
        counts.append(pos.n)
        assert pos.footprint() == a["positions_bytes_g8"][s], s
        assert yp.footprint() == a["yp_bytes_g8"][s], s
        total += ms.u64(ms.agg_sum(yp))
        if s == 0:  # the shard's first positions are global row ids of shard 0
            check_sampled_positions(ms, pos, lambda mm, ss: synth.gen_host("c5.X", mm, ss), O.LT, 1 << 16,
                                    samples=((0, 1 << 18),))
        del X, Y, pos, yp
    assert counts == a["shard_counts_g8"]
    offs = D.exclusive_offsets(counts)
    assert offs[0] == 0 and offs[1] == a["shard_counts_g8"][0] and offs[-1] + counts[-1] == a["count"]
    assert total % (1 << 64) == a["sum_projected"]


# ------------------------------------------------------------------ sharded c2 / c4
@pytest.mark.parametrize("G", [3])
def test_c2_sharded_full(G):
    """BJ.c2 cut into G row-range shards (D-18), one after another on one GPU:
    the C1 counts and the C2 sums combine to the full-size anchors."""
    ms = get_ms()
    from paper_2004_09350_b200 import dist as D
    a = anchors()["c2"]
    n = a["n"]
    count, total = 0, 0
    for s in range(G):
        start, end = D.shard_range(n, G, s)
        X, Y, pos, yp, yu = c2_chain(ms, end - start, start)
        count += pos.n
        total += ms.u64(ms.agg_sum(yp))
        assert ms.u64(ms.agg_sum(yp)) == ms.u64(ms.agg_sum(yu))
        del X, Y, pos, yp, yu
    assert count == a["count"]
    assert total % (1 << 64) == a["sum_projected"]


@pytest.mark.parametrize("G", [4])
def test_c4_sharded_full(G):
    """BJ.c4's D-16 chain on G row-range shards: the per-shard 1000-group sums
    added element-wise (the C3 allreduce of SURVEY.md §8(e)) equal the anchors."""
    ms = get_ms()
    from paper_2004_09350_b200 import dist as D
    a = anchors()["c4"]
    n = a["n"]
    g1 = np.zeros(1000, np.uint64)
    g2 = np.zeros(1000, np.uint64)
    c1 = c2 = 0
    for s in range(G):
        start, end = D.shard_range(n, G, s)
        g = c4_chain(ms, end - start, start)
        g1 += g["g1"]
        g2 += g["g2"]
        c1 += g["pos1"].n
        c2 += g["pos2"].n
        del g
    assert c1 == a["count_pos1"] and c2 == a["count_pos2"]
    assert [int(x) for x in g1] == a["grouped_m1"]
    assert [int(x) for x in g2] == a["grouped_m2"]


# ------------------------------------------------------------------ K7: fused semi-join (D-16)
def test_c4_semijoin_fused_reduced():
    """ms_semijoin (gather k1 at pos1 in shared memory, bitmap test, surviving
    ranks, pos1 at those ranks) is byte-identical to the oracle's operator-at-a-time
    D-16 chain pos2 = project(pos1, select(project(k1, pos1), IN_BITMAP)); the
    non-fused fallback (keys without O(1) access) gives the same bytes."""
    ms = get_ms()
    n = 1 << 22
    D4 = synth.D4
    bm_host = synth.bitmap_c4()
    bm = to_torch(bm_host)
    k0 = ms.compress(dev("c4.k0", n), ms.static_bp(12))
    k1 = ms.compress(dev("c4.k1", n), ms.static_bp(18))
    pos1 = ms.select(k0, ms.BETWEEN, 0, 365, out_fmt=ms.delta_bp(512))
    ok0 = O.encode(synth.gen_host("c4.k0", n), O.STATIC_BP, 12)
    ok1 = O.encode(synth.gen_host("c4.k1", n), O.STATIC_BP, 18)
    opos1 = O.select(ok0, O.BETWEEN, 0, 365, out_fmt=O.DELTA_BP, out_block=512)
    oidx = O.select(O.project(ok1, opos1, 0, O.STATIC_BP, 18, 0), O.IN_BITMAP, bitmap=bm_host, bitmap_bits=D4[1],
                    out_fmt=O.DELTA_BP, out_block=512)
    for fo in (ms.delta_bp(512), ms.uncompr()):
        opos2 = O.project(opos1, oidx, 0, *oracle_fmt(fo))
        assert_same_image(ms.semijoin(k1, pos1, bm, D4[1], out_fmt=fo), opos2, f"K7 fused -> {fo}")
    k1d = ms.morph(k1, ms.delta_bp(2048))  # no O(1) row access: the operator chain
    opos2 = O.project(opos1, oidx, 0, O.DELTA_BP, 0, 512)
    assert_same_image(ms.semijoin(k1d, pos1, bm, D4[1]), opos2, "K7 fallback chain")


def test_c4_semijoin_fused_full():
    ms = get_ms()
    a = anchors()["c4"]
    n = a["n"]
    bm = to_torch(synth.bitmap_c4())
    k0 = ms.compress(dev("c4.k0", n), ms.static_bp(12))
    k1 = ms.compress(dev("c4.k1", n), ms.static_bp(18))
    pos1 = ms.select(k0, ms.BETWEEN, 0, 365, out_fmt=ms.delta_bp(512))
    pos2 = ms.semijoin(k1, pos1, bm, synth.D4[1])
    assert pos2.n == a["count_pos2"]
    assert pos2.footprint() == a["pos2_bytes"]
