"""Error behaviour of the C ABI on malformed inputs (include/ms.h; SPEC.md
S:127 CorruptBody, S:59/290 IndexOutOfRange): corrupt RLE bodies, positions
outside the data, malformed host width tables. Every case must come back as a
status code — never as an out-of-bounds access (the process stays usable and
later ops still give oracle-exact results)."""
import numpy as np
import pytest

import oracle as O
from tests.gpu_util import assert_same_image, get_ms, to_torch

pytestmark = pytest.mark.gpu

CORRUPT, RANGE = 5, 4


@pytest.mark.parametrize("runs", [
    [(3, 2), (7, 1 << 63), (9, 3)],                    # one huge length: total mismatch, run ends past n
    [(3, 2), (7, (1 << 64) - 2), (9, 5)],              # lengths wrapping mod 2^64 to the right total
    [(3, 0), (7, 5)],                                  # zero length
])
def test_corrupt_rle_select_and_morph(runs):
    ms = get_ms()
    pay = np.array([x for vl in runs for x in vl], np.uint64)
    n = 5
    col = ms.Column.from_host(ms.rle(), n, pay, n_runs=len(runs))
    with pytest.raises(ms.MsError) as e:
        ms.select(col, ms.GE, 0, out_fmt=ms.delta_bp(512))
    assert e.value.code == CORRUPT
    with pytest.raises(ms.MsError) as e:
        ms.morph(col, ms.delta_bp(128))
    assert e.value.code == CORRUPT
    with pytest.raises(ms.MsError) as e:
        ms.agg_sum(col, check=True)
    assert e.value.code == CORRUPT
    # the device is still healthy: a valid op afterwards is oracle-exact
    v = np.arange(3000, dtype=np.uint64) % 7
    c = ms.compress(to_torch(v), ms.dyn_bp(128))
    assert_same_image(c, O.encode(v, O.DYN_BP, 0, 128), "after corrupt input")


def test_agg_sum_positions_out_of_range():
    ms = get_ms()
    v = np.arange(1000, dtype=np.uint64)
    data = ms.compress(to_torch(v), ms.for_bp(128))
    pos = ms.compress(to_torch(np.array([1, 5, 1000], np.uint64)), ms.uncompr())
    with pytest.raises(ms.MsError) as e:
        ms.agg_sum(data, pos, check=True)
    assert e.value.code == RANGE
    ms.check_errors()  # the sticky word was cleared by the read
    pos_ok = ms.compress(to_torch(np.array([1, 5, 999], np.uint64)), ms.uncompr())
    assert ms.u64(ms.agg_sum(data, pos_ok, check=True)) == 1 + 5 + 999


def test_agg_sum_grouped_range_check():
    ms = get_ms()
    g = ms.compress(to_torch(np.array([0, 1, 7], np.uint64)), ms.uncompr())
    v = ms.compress(to_torch(np.array([1, 2, 3], np.uint64)), ms.uncompr())
    with pytest.raises(ms.MsError) as e:
        ms.agg_sum_grouped(g, v, 4, check=True)
    assert e.value.code == RANGE


@pytest.mark.parametrize("bad", ["wide", "decreasing", "payload", "cw0"])
def test_column_to_device_validates_width_table(bad):
    ms = get_ms()
    v = np.arange(1024, dtype=np.uint64) * 3
    oc = O.encode(v, O.DYN_BP, 0, 128)
    cw, pay = oc.cw.copy(), oc.payload.copy()
    if bad == "wide":
        cw[2:] += 70
        pay = np.zeros(int(cw[-1]) * 2, np.uint64)
    elif bad == "decreasing":
        cw[3] = cw[2] - 1
    elif bad == "payload":
        pay = pay[:-2]
    else:
        cw = cw + 1
    with pytest.raises(ms.MsError) as e:
        ms.Column.from_host(ms.dyn_bp(128), 1024, pay, cw=cw, rem=oc.rem)
    assert e.value.code == CORRUPT
    good = ms.Column.from_host(ms.dyn_bp(128), 1024, oc.payload, cw=oc.cw, rem=oc.rem)
    assert_same_image(good, oc, "valid upload")


def test_release_on_other_stream():
    """A column created on one stream and read on another is released only after
    the reader's work (the creating stream waits on it): results stay exact."""
    import torch
    ms = get_ms()
    s2 = torch.cuda.Stream()
    v = np.arange(1 << 20, dtype=np.uint64) % 1000
    expect = O.decode(O.select(O.encode(v, O.UNCOMPR), O.LT, 100, out_fmt=O.UNCOMPR))
    for _ in range(3):
        X = ms.compress(to_torch(v), ms.static_bp(10))
        s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s2):
            pos = ms.select(X, ms.LT, 100, out_fmt=ms.delta_bp(512), stream=s2)
        del X
        junk = torch.full((1 << 22,), -1, dtype=torch.int64, device="cuda")  # may reuse X's block
        torch.cuda.current_stream().wait_stream(s2)
        got = ms.to_u64_numpy(ms.decompress(pos))
        assert np.array_equal(got, expect)
        del junk


@pytest.mark.parametrize("kind", ["unsorted", "duplicate", "across_blocks"])
def test_semijoin_rejects_unsorted_positions(kind):
    """ms_semijoin requires strictly increasing positions (include/ms.h): the
    fused kernel flags MS_E_INVALID for a block that is not, or whose successor
    does not start after it; sorted positions in the same formats stay exact."""
    import torch
    ms = get_ms()
    rng = np.random.default_rng(11)
    n = 20_000
    keys = rng.integers(0, 1000, n).astype(np.uint64)
    K = ms.compress(to_torch(keys), ms.static_bp(10))
    bm = np.zeros(16, np.uint64)
    bm[:8] = 0x5555555555555555
    bmt = torch.from_numpy(bm.view(np.int64)).cuda()
    p = np.sort(rng.choice(n, 3000, replace=False)).astype(np.uint64)
    bad = p.copy()
    if kind == "unsorted":
        bad[10], bad[11] = bad[11], bad[10]
    elif kind == "duplicate":
        bad[100] = bad[99]
    else:  # block 1 starts before block 0 ends
        bad[512] = bad[511] - 1 if bad[511] - 1 > bad[510] else bad[511]
    P = ms.compress(to_torch(bad), ms.uncompr())
    with pytest.raises(ms.MsError) as e:
        ms.semijoin(K, P, bmt, 1000)
    assert e.value.code == 1  # MS_E_INVALID
    good = ms.compress(to_torch(p), ms.uncompr())
    got = ms.to_u64_numpy(ms.decompress(ms.semijoin(K, good, bmt, 1000, out_fmt=ms.uncompr())))
    keep = (keys[p.astype(np.int64)] < 512) & (keys[p.astype(np.int64)] % 2 == 0)
    assert np.array_equal(got, p[keep])
