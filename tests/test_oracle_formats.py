"""Oracle pins: the five formats + UNCOMPR and the column layout (PAPER.md
P:108-126, 420-421, 433-440; readings D-1..D-9 in DESIGN.md).
Pinned by worked examples, closed-form size laws, brute-force round trips over
edge lengths and an independent numpy/big-int construction of each image."""
import numpy as np
import pytest

import oracle as O
from tests.conftest import as_int
from tests.test_oracle_bitpack import bigint_pack

RNG = np.random.default_rng(99)
BLOCKS = (128, 256, 512, 1024, 2048)
M64 = (1 << 64) - 1


def dyn_values():
    return np.concatenate([np.zeros(128, np.uint64), np.full(128, 3, np.uint64),
                           np.full(128, 1 << 63, np.uint64), np.tile(np.array([1, 2], np.uint64), 64),
                           np.array([7, 7, 7], np.uint64)])


def test_dynbp_worked_example(worked):
    ex = worked["dyn_bp"]
    c = O.encode(dyn_values(), O.DYN_BP, 0, ex["block"])
    assert list(np.diff(c.cw.astype(np.int64))) == ex["widths"]
    assert list(c.cw) == ex["cw"]
    assert c.payload_words == ex["payload_words"]
    assert list(c.rem) == ex["rem"]
    assert c.n_blocks == 4 and c.n_rem == 3
    # size law (closed form): sum B*w_b/8 + 4(nb+1) + 8*rem
    assert c.footprint() == sum(128 * w // 8 for w in ex["widths"]) + 4 * 5 + 8 * 3


def test_delta_worked_example(worked):
    ex = worked["delta_bp"]
    v = np.arange(*ex["values_range"], dtype=np.uint64)
    c = O.encode(v, O.DELTA_BP, 0, ex["block"])
    assert list(c.ref) == ex["ref"] and list(c.cw) == ex["cw"]
    assert [int(x) for x in c.payload] == [as_int(x) for x in ex["payload"]]


def test_delta_decreasing_wraps_to_64_bits():
    # a decreasing sequence round-trips via mod-2^64 wrap-around; deltas need 64 bits
    v = np.arange(1000, 1000 - 128, -1).astype(np.uint64)
    c = O.encode(v, O.DELTA_BP, 0, 128)
    assert list(c.cw) == [0, 64]
    assert np.array_equal(O.decode(c), v)


def test_for_worked_example(worked):
    ex = worked["for_bp"]
    v = (1000 + np.arange(128) % 7).astype(np.uint64)
    c = O.encode(v, O.FOR_BP, 0, ex["block"])
    assert list(c.ref) == ex["ref"] and list(c.cw) == ex["cw"]
    assert c.payload_words == ex["payload_words"]
    assert int(c.payload[0]) == as_int(ex["payload0"])


def test_for_constant_block_zero_width():
    # constant FOR block -> w = 0, no payload
    c = O.encode(np.full(128, 7, np.uint64), O.FOR_BP, 0, 128)
    assert list(c.cw) == [0, 0] and c.payload_words == 0 and list(c.ref) == [7]
    assert np.array_equal(O.decode(c), np.full(128, 7, np.uint64))


def test_rle_worked_example(worked):
    ex = worked["rle"]
    c = O.encode(ex["values"], O.RLE)
    assert [int(x) for x in c.payload] == ex["payload"] and c.n_runs == 3
    assert list(O.decode(c)) == ex["values"]


def test_column_split(worked):
    ex = worked["column_split"]
    c = O.encode(RNG.integers(0, 1000, ex["n"]).astype(np.uint64), O.DYN_BP, 0, ex["block"])
    assert (c.n_blocks, c.n_rem) == (ex["n_blocks"], ex["n_rem"])


def independent_image(v, fmt, B):
    """Block-format image built with numpy reductions + big-int packing (an independent
    formulation of D-4..D-6), for comparison with the oracle's bit loops."""
    v = [int(x) for x in v]
    nb = len(v) // B
    cw, ref, payload = [0], [], []
    for b in range(nb):
        x = v[b * B:(b + 1) * B]
        if fmt == O.FOR_BP:
            r = min(x); codes = [xi - r for xi in x]; ref.append(r)
        elif fmt == O.DELTA_BP:
            codes = [0] + [(x[j] - x[j - 1]) & M64 for j in range(1, B)]; ref.append(x[0])
        else:
            codes = x
        w = max(codes).bit_length()
        cw.append(cw[-1] + w)
        if w:
            payload += bigint_pack(codes, w)
    return cw, ref, payload, v[nb * B:]


def rand_column(n, kind):
    if kind == "small":
        return RNG.integers(0, 64, n).astype(np.uint64)
    if kind == "wide":
        return RNG.integers(0, 2**64 - 1, n, dtype=np.uint64, endpoint=True)
    if kind == "sorted":
        return np.sort(RNG.integers(1 << 47, (1 << 47) + 100_000, n)).astype(np.uint64)
    if kind == "runs":
        return np.repeat(RNG.integers(0, 5, max(1, n // 7 + 1)), 7)[:n].astype(np.uint64)
    if kind == "outlier":
        x = RNG.integers(0, 64, n).astype(np.uint64)
        x[RNG.random(n) < 0.01] = (1 << 63) - 1
        return x
    raise ValueError(kind)


@pytest.mark.parametrize("fmt", [O.DYN_BP, O.FOR_BP, O.DELTA_BP])
@pytest.mark.parametrize("B", BLOCKS)
def test_block_formats_against_independent_image(fmt, B):
    for kind in ("small", "wide", "sorted", "outlier"):
        for n in (0, 1, B - 1, B, B + 1, 3 * B + 7):
            v = rand_column(n, kind)
            c = O.encode(v, fmt, 0, B)
            cw, ref, payload, rem = independent_image(v, fmt, B)
            assert list(c.cw) == cw
            assert [int(x) for x in c.ref] == (ref if fmt != O.DYN_BP else [])
            assert [int(x) for x in c.payload] == payload
            assert [int(x) for x in c.rem] == rem
            assert np.array_equal(O.decode(c), v)
            # footprint closed form (SURVEY c.2)
            nb = n // B
            fp = 8 * len(payload) + 4 * (nb + 1) + 8 * (n - nb * B) + (8 * nb if fmt != O.DYN_BP else 0)
            assert c.footprint() == fp


@pytest.mark.parametrize("kind", ["small", "wide", "sorted", "runs", "outlier"])
def test_roundtrip_all_formats(kind):
    for n in (0, 1, 127, 128, 129, 2048 * 3 + 5):
        v = rand_column(n, kind)
        specs = [(O.UNCOMPR, 0, 0), (O.RLE, 0, 0), (O.STATIC_BP, 0, 0), (O.STATIC_BP, 64, 0)]
        specs += [(f, 0, B) for f in (O.DYN_BP, O.FOR_BP, O.DELTA_BP) for B in (128, 2048)]
        for f, w, B in specs:
            c = O.encode(v, f, w, B)
            assert np.array_equal(O.decode(c), v), (f, w, B, n)


def test_static_auto_width_and_explicit():
    v = np.array([0, 5, 1023], np.uint64)
    c = O.encode(v, O.STATIC_BP, 0)
    assert c.bit_width == 10 and c.payload_words == 1
    assert [int(x) for x in c.payload] == bigint_pack([0, 5, 1023], 10)
    z = O.encode(np.zeros(5, np.uint64), O.STATIC_BP, 0)
    assert z.bit_width == 1  # max(1, ebw(0))
    c = O.encode(np.zeros(0, np.uint64), O.DYN_BP, 0, 512)
    assert list(c.cw) == [0] and c.footprint() == 4  # D-14


def test_rle_maximal_runs_identity():
    v = rand_column(5000, "runs")
    c = O.encode(v, O.RLE)
    vals, lens = c.payload[0::2], c.payload[1::2]
    assert int(lens.sum()) == v.size and (lens >= 1).all()
    assert (vals[1:] != vals[:-1]).all()  # maximal: adjacent runs differ
    assert np.array_equal(np.repeat(vals, lens.astype(np.int64)), v)


def test_uncompr_image_is_values():
    v = rand_column(100, "wide")
    c = O.encode(v, O.UNCOMPR)
    assert np.array_equal(c.payload, v) and c.footprint() == 800


def test_invalid_block_size():
    with pytest.raises(O.OracleError):
        O.encode(np.zeros(10, np.uint64), O.DYN_BP, 0, 100)
