#!/usr/bin/env python3
"""Full-size regression anchors for BASELINE.json configs c2..c5, computed by the
CPU oracle ONLY (oracle/ + the seeded generators of synth/), written to
tests/golden/config_anchors.json. The GPU tests compare the CUDA path against
these at full size (counts, sums, grouped sums, per-shard counts); byte-exact
image parity is checked at reduced sizes where the oracle runs in seconds.

Each config is cut into row shards of 2^24 (multiples of every block size);
select counts and sums are additive over shards, so every anchor is an exact
property of the full column. usage: python tools/make_anchors.py [c2 c3 c4 c5]
"""
from __future__ import annotations

import json
import os
import sys
import time
from multiprocessing import Pool

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import synth  # noqa: E402

SHARD = 1 << 24
M64 = (1 << 64) - 1
OUT = os.path.join(ROOT, "tests", "golden", "config_anchors.json")


def shards(n):
    return [(s, min(SHARD, n - s)) for s in range(0, n, SHARD)]


# ---------------------------------------------------------------- c2
def c2_shard(arg):
    start, m = arg
    X = O.encode(synth.gen_host("c2.X", m, start), O.DYN_BP, 0, 512)
    Y = O.encode(synth.gen_host("c2.Y", m, start), O.FOR_BP, 0, 512)
    pos = O.select(X, O.EQ, 17, row_offset=start, out_fmt=O.DELTA_BP, out_block=512)
    yp = O.project(Y, pos, start, O.FOR_BP, 0, 512)
    return pos.n, O.agg_sum(yp), O.decode(pos), O.decode(yp)


def image_bytes(values, fmt, block):
    """Footprint of the oracle's canonical image of `values`."""
    return O.encode(values, fmt, 0, block).footprint()


# ---------------------------------------------------------------- c5
def c5_shard(arg):
    start, m = arg
    X = O.encode(synth.gen_host("c5.X", m, start), O.DYN_BP, 0, 512)
    Y = O.encode(synth.gen_host("c5.Y", m, start), O.FOR_BP, 0, 512)
    pos = O.select(X, O.LT, 1 << 16, row_offset=start, out_fmt=O.DELTA_BP, out_block=512)
    yp = O.project(Y, pos, start, O.FOR_BP, 0, 512)
    return pos.n, O.agg_sum(yp), O.decode(pos), O.decode(yp)


def c5_images(res, G):
    """Footprints of the positions (DELTA_BP{512}) and Y' (FOR_BP{512}) images
    when the 2^32 rows are cut into G row-range shards (2^24-row pieces in order;
    G divides 256): per-shard images, encoded from the concatenated decoded
    pieces of each shard."""
    per = len(res) // G
    pos_b, yp_b = [], []
    for k in range(G):
        part = res[k * per:(k + 1) * per]
        pos_b.append(image_bytes(np.concatenate([r[2] for r in part]), O.DELTA_BP, 512))
        yp_b.append(image_bytes(np.concatenate([r[3] for r in part]), O.FOR_BP, 512))
    return pos_b, yp_b


# ---------------------------------------------------------------- c4 (D-16 chain)
def c4_shard(arg):
    start, m = arg
    D = synth.D4
    bm = synth.bitmap_c4()
    gattr = O.encode(synth.gen_host("c4.gattr", D[3]), O.STATIC_BP, 10)
    k0 = O.encode(synth.gen_host("c4.k0", m, start), O.STATIC_BP, 12)
    k1 = O.encode(synth.gen_host("c4.k1", m, start), O.STATIC_BP, 18)
    k3 = O.encode(synth.gen_host("c4.k3", m, start), O.STATIC_BP, 17)
    m1 = O.encode(synth.gen_host("c4.m1", m, start), O.DYN_BP, 0, 512)
    m2 = O.encode(synth.gen_host("c4.m2", m, start), O.DYN_BP, 0, 512)
    pos1 = O.select(k0, O.BETWEEN, 0, 365, row_offset=start, out_fmt=O.DELTA_BP, out_block=512)
    k1p = O.project(k1, pos1, start, O.STATIC_BP, 18, 0)
    idx = O.select(k1p, O.IN_BITMAP, bitmap=bm, bitmap_bits=D[1], out_fmt=O.DELTA_BP, out_block=512)
    pos2 = O.project(pos1, idx, 0, O.DELTA_BP, 0, 512)
    m1p = O.project(m1, pos2, start, O.DYN_BP, 0, 512)
    m2p = O.project(m2, pos2, start, O.DYN_BP, 0, 512)
    k3p = O.project(k3, pos2, start, O.STATIC_BP, 17, 0)
    gid = O.project(gattr, k3p, 0, O.STATIC_BP, 10, 0)
    g1 = O.agg_sum_grouped(gid, m1p, 1000)
    g2 = O.agg_sum_grouped(gid, m2p, 1000)
    return pos1.n, pos2.n, O.agg_sum(m1p), O.agg_sum(m2p), g1, g2, O.decode(pos1), O.decode(pos2)


def run_c4(pool):
    n = 600_000_000
    res = pool.map(c4_shard, shards(n))
    g1 = np.zeros(1000, np.uint64)
    g2 = np.zeros(1000, np.uint64)
    for r in res:
        g1 += r[4]
        g2 += r[5]
    return {"n": n, "count_pos1": sum(r[0] for r in res), "count_pos2": sum(r[1] for r in res),
            "sum_m1": sum(r[2] for r in res) & M64, "sum_m2": sum(r[3] for r in res) & M64,
            "bitmap_bits_set": int(sum(bin(int(w)).count("1") for w in synth.bitmap_c4())),
            "grouped_m1": [int(x) for x in g1], "grouped_m2": [int(x) for x in g2],
            "pos1_bytes": image_bytes(np.concatenate([r[6] for r in res]), O.DELTA_BP, 512),
            "pos2_bytes": image_bytes(np.concatenate([r[7] for r in res]), O.DELTA_BP, 512)}


# ---------------------------------------------------------------- c3 (whole column)
def run_c3():
    n = 1 << 29
    x = synth.gen_host("c3.x", n)
    runs = int(np.count_nonzero(np.diff(x))) + 1
    lo, hi = 10**6, 2 * 10**6
    r = O.encode(x, O.RLE)
    d = O.encode(x, O.DELTA_BP, 0, 2048)
    pos_r = O.select(r, O.BETWEEN, lo, hi, out_fmt=O.DELTA_BP, out_block=512)
    pos_d = O.select(d, O.BETWEEN, lo, hi, out_fmt=O.DELTA_BP, out_block=512)
    assert pos_r.n == pos_d.n
    pv = O.decode(pos_d)
    s_r = O.agg_sum(r, pos_r)
    s_d = O.agg_sum(d, pos_d)
    assert s_r == s_d
    sbp = O.morph(d, O.STATIC_BP, 0, 0)
    return {"n": n, "runs": runs, "rle_runs": r.n_runs, "max": int(x.max()), "static_bp_auto_width": sbp.bit_width,
            "sum_all": int(O.agg_sum(d)), "count": int(pos_d.n), "first": int(pv[0]) if pv.size else None,
            "last": int(pv[-1]) if pv.size else None, "sum_selected": int(s_d),
            "delta_bp2048_payload_bytes": int(8 * d.payload.size), "positions_bytes": pos_d.footprint()}


def main():
    which = sys.argv[1:] or ["c2", "c3", "c4", "c5"]
    anchors = json.load(open(OUT)) if os.path.exists(OUT) else {}
    anchors["_about"] = ("Full-size anchors of BASELINE.json configs, computed by tools/make_anchors.py from "
                         "oracle/ only (shards of 2^24 rows; counts and sums are additive).")
    with Pool(min(8, os.cpu_count() or 1)) as pool:
        if "c2" in which:
            t = time.time()
            res = pool.map(c2_shard, shards(1 << 28))
            yv = np.concatenate([r[3] for r in res])
            anchors["c2"] = {"n": 1 << 28, "count": sum(r[0] for r in res),
                             "sum_projected": sum(r[1] for r in res) & M64,
                             "positions_bytes": image_bytes(np.concatenate([r[2] for r in res]), O.DELTA_BP, 512),
                             "yp_for_bytes": image_bytes(yv, O.FOR_BP, 512),
                             "yp_uncompr_bytes": 8 * int(yv.size)}
            print("c2", anchors["c2"], f"{time.time() - t:.0f}s", flush=True)
        if "c5" in which:
            t = time.time()
            res = pool.map(c5_shard, shards(1 << 32))
            per8 = [sum(r[0] for r in res[k * 32:(k + 1) * 32]) for k in range(8)]
            p1, y1 = c5_images(res, 1)
            p8, y8 = c5_images(res, 8)
            anchors["c5"] = {"n": 1 << 32, "count": sum(r[0] for r in res),
                             "sum_projected": sum(r[1] for r in res) & M64, "shard_counts_g8": per8,
                             "positions_bytes": p1[0], "yp_bytes": y1[0],
                             "positions_bytes_g8": p8, "yp_bytes_g8": y8}
            print("c5", anchors["c5"], f"{time.time() - t:.0f}s", flush=True)
        if "c4" in which:
            t = time.time()
            anchors["c4"] = run_c4(pool)
            print("c4", {k: v for k, v in anchors["c4"].items() if not k.startswith("grouped")},
                  f"{time.time() - t:.0f}s", flush=True)
    if "c3" in which:
        t = time.time()
        anchors["c3"] = run_c3()
        print("c3", anchors["c3"], f"{time.time() - t:.0f}s", flush=True)
    with open(OUT, "w") as f:
        json.dump(anchors, f, indent=1)


if __name__ == "__main__":
    main()
