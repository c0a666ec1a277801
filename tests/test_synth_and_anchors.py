"""Input generator pins (synth/) and the oracle on BASELINE.json configs[0] (c1).

The c1 numbers are SURVEY.md §8(c) c.4 regression anchors (computed there by a
numpy script and re-derived by an independent scalar C program); the oracle
must land on them exactly."""
import numpy as np

import oracle as O
import synth
from tests.conftest import as_int


def test_splitmix64_vector(worked):
    ex = worked["splitmix64"]
    # R(s, 0) is splitmix64(s)'s first output
    r = synth.recipe(synth.SYN_MASK, seed=ex["seed"], mask=(1 << 64) - 1)
    assert int(synth.gen_host(r, 1)[0]) == as_int(ex["first"])


def test_c1_first_values(worked):
    assert [int(x) for x in synth.gen_host("c1.X", 8)] == worked["c1_first_values"]["values"]


def test_counter_based_sharding_invariance():
    # any split of the rows gives identical values (needed for row-range sharding, §8(e))
    for name in ("c2.X", "c3.x", "c4.k1", "C2.X", "c5.Y"):
        full = synth.gen_host(name, 10_000)
        parts = np.concatenate([synth.gen_host(name, 3_000, 0), synth.gen_host(name, 4_000, 3_000),
                                synth.gen_host(name, 3_000, 7_000)])
        assert np.array_equal(full, parts), name


def test_c3_generator_shape():
    x = synth.gen_host("c3.x", 1 << 16)
    d = np.diff(x.astype(np.int64))
    assert x[0] == 0 and (d >= 0).all() and d.max() <= 16
    runs = 1 + np.count_nonzero(d)
    assert 700 < runs < 1400  # geometric run lengths, mean 64 -> ~1024 runs


def test_c1_anchors():
    """configs[0]: select(X sBP10, LT 102) -> DELTA_BP{512}; sum of X at the positions."""
    X = synth.gen_host("c1.X", 1 << 20)
    xc = O.encode(X, O.STATIC_BP, 10)
    assert xc.footprint() == 1_310_720
    pos = O.select(xc, O.LT, 102, out_fmt=O.DELTA_BP, out_block=512)
    assert pos.n == 104_227
    assert pos.footprint() == 88_864
    assert (pos.n_blocks, pos.n_rem) == (203, 291)
    w = np.diff(pos.cw.astype(np.int64))
    assert (np.count_nonzero(w == 6), np.count_nonzero(w == 7)) == (107, 96)
    assert O.agg_sum(xc, pos) == 5_277_336
    assert O.agg_sum(O.project(xc, pos, 0, O.UNCOMPR)) == 5_277_336


def test_full_size_anchor_file_matches_survey():
    """tests/golden/config_anchors.json is written by tools/make_anchors.py from
    oracle/ only; its image sizes must equal the numbers SURVEY.md §8(a) a5/a6
    and §8(e) print (computed there by two independent scripts, a numpy one and
    a scalar C one). Agreement pins the anchors the -m gpu tests assert."""
    import json
    import os
    p = os.path.join(os.path.dirname(__file__), "golden", "config_anchors.json")
    a = json.load(open(p))
    assert a["c2"]["positions_bytes"] == 1_476_652 and a["c2"]["yp_for_bytes"] == 2_624_044
    assert a["c4"]["pos1_bytes"] == 66_462_044 and a["c4"]["pos2_bytes"] == 4_719_624
    c5 = a["c5"]
    assert c5["positions_bytes"] == 245_585_644 and c5["yp_bytes"] == 677_386_156
    assert sum(c5["positions_bytes_g8"]) == 245_606_552 and sum(c5["yp_bytes_g8"]) == 677_397_400
    assert c5["positions_bytes_g8"][0] == 30_699_776 and c5["yp_bytes_g8"][0] == 84_678_464
    assert c5["shard_counts_g8"] == [33_556_227, 33_555_886, 33_555_972, 33_546_492, 33_560_502, 33_550_630,
                                     33_557_332, 33_553_873]
    assert c5["count"] == 268_436_914 and c5["sum_projected"] == 409_182_112_845_958
    assert a["c3"]["delta_bp2048_payload_bytes"] == 326_463_488 and a["c3"]["static_bp_auto_width"] == 27
