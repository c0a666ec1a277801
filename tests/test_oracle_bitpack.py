"""Oracle pins: null suppression / static bit packing (
SPEC.md S:23-94). Checked against SPEC's worked examples, the paper's Table
widths and an independent big-integer construction of the LSB-first stream."""
import numpy as np
import pytest

import oracle as O
from tests.conftest import as_int

RNG = np.random.default_rng(1234)


def bigint_pack(values, w):
    """Independent formulation of the LSB-first stream: the stream is the integer
    sum_i v_i * 2^(i*w); word k is bits [64k, 64k+64) of that integer."""
    acc = 0
    for i, v in enumerate(values):
        acc |= int(v) << (i * w)
    nwords = (len(values) * w + 63) // 64
    return [(acc >> (64 * k)) & ((1 << 64) - 1) for k in range(nwords)]


def test_pack_worked_examples(worked):
    for ex in worked["pack"]:
        vals = [as_int(x) for x in ex["values"]]
        got = [int(x) for x in O.pack(vals, ex["w"])]
        assert got == [as_int(x) for x in ex["words"]], ex["cite"]


def test_get_at_worked_examples(worked):
    for ex in worked["get_at"]:
        words = O.pack(ex["values"], ex["w"])
        assert O.get_at(words, ex["w"], ex["i"]) == ex["expected"], ex["cite"]


def test_ebw_examples(worked):
    for ex in worked["ebw"]:
        assert O.ebw(as_int(ex["v"])) == ex["expected"], ex["cite"]


def test_ebw_closed_form():
    # ebw(v) = floor(log2 v) + 1 = Python's int.bit_length()
    for v in [0, 1, 2, 3, 4, 255, 256, (1 << 63) - 1, 1 << 63, (1 << 64) - 1]:
        assert O.ebw(v) == int(v).bit_length()
    for v in RNG.integers(0, 2**63, 200, dtype=np.uint64):
        for s in (0, 1, 17, 40):
            x = int(v) >> s
            assert O.ebw(x) == x.bit_length()


@pytest.mark.parametrize("w", list(range(1, 65)))
def test_pack_roundtrip_all_widths(w):
    for n in (0, 1, 63, 64, 65, int(RNG.integers(100, 3000))):
        hi = (1 << w) - 1
        vals = [int(x) & hi for x in RNG.integers(0, 2**64 - 1, n, dtype=np.uint64, endpoint=True)]
        words = O.pack(vals, w)
        # size law: 8 * ceil(n*w/64) bytes
        assert words.size == (n * w + 63) // 64
        assert [int(x) for x in words] == bigint_pack(vals, w)
        back = O.unpack(words, n, w)
        assert [int(x) for x in back] == vals
        for i in range(0, n, max(1, n // 17)):
            assert O.get_at(words, w, i) == vals[i]


def test_width_overflow():
    with pytest.raises(O.OracleError) as e:
        O.pack([4], 2)
    assert e.value.code == O.E_WIDTH_OVERFLOW
    with pytest.raises(O.OracleError):
        O.encode([1, 2, 300], O.STATIC_BP, 8)


def test_order_preservation_static_codes():
    # for a < b the packed codes compare a < b (codes are the values themselves)
    w = 13
    vals = sorted(int(x) for x in RNG.integers(0, 1 << w, 500))
    words = O.pack(vals, w)
    codes = [O.get_at(words, w, i) for i in range(len(vals))]
    assert codes == vals


def test_padding_bits_zero():
    # D-2: unused high bits of the last word are zero
    words = O.pack([(1 << 7) - 1] * 3, 7)  # 21 bits used
    assert int(words[0]) == (1 << 21) - 1
