"""Helpers shared by the GPU parity tests: run the same seeded input through
the CUDA path (paper_2004_09350_b200.ms, via the C ABI) and through the oracle
(oracle/, plain C), and compare images section by section."""
import numpy as np

import oracle as O

ms = None


def get_ms():
    global ms
    if ms is None:
        from paper_2004_09350_b200 import ms as _ms
        ms = _ms
    return ms


def to_torch(values: np.ndarray):
    import torch
    v = np.ascontiguousarray(values, dtype=np.uint64)
    return torch.from_numpy(v.view(np.int64).copy()).cuda()


def oracle_fmt(f):
    """ms.Fmt -> (oracle format, bit_width, block_size); numeric codes are the
    normative ones of DESIGN.md §3 on both sides, mapped here by name."""
    m = get_ms()
    code = {m.UNCOMPR: O.UNCOMPR, m.STATIC_BP: O.STATIC_BP, m.DYN_BP: O.DYN_BP, m.DELTA_BP: O.DELTA_BP,
            m.FOR_BP: O.FOR_BP, m.RLE: O.RLE}[f.format]
    return code, f.bit_width, f.block_size


def oracle_op(op):
    m = get_ms()
    return {m.EQ: O.EQ, m.NE: O.NE, m.LT: O.LT, m.LE: O.LE, m.GT: O.GT, m.GE: O.GE, m.BETWEEN: O.BETWEEN,
            m.IN_BITMAP: O.IN_BITMAP}[op]


def assert_same_image(gpu_col, ocol, what=""):
    """Bit-exact: descriptor fields and the bytes of every image section."""
    m = get_ms()
    assert gpu_col.n == ocol.n, (what, gpu_col.n, ocol.n)
    assert gpu_col.n_blocks == ocol.n_blocks and gpu_col.n_rem == ocol.n_rem, what
    if ocol.format == O.STATIC_BP:
        assert gpu_col.fmt.bit_width == ocol.bit_width, (what, gpu_col.fmt, ocol.bit_width)
    if ocol.format == O.RLE:
        assert gpu_col.n_runs == ocol.n_runs, what
    img = gpu_col.images()
    for sec in ("payload", "cw", "ref", "rem"):
        g, o = img[sec], getattr(ocol, sec)
        assert g.size == o.size, (what, sec, g.size, o.size)
        if not np.array_equal(g, o):
            bad = np.nonzero(g != o)[0][:5]
            raise AssertionError(f"{what}: section {sec} differs at {bad.tolist()} "
                                 f"gpu={g[bad].tolist()} oracle={o[bad].tolist()}")
    assert gpu_col.footprint() == ocol.footprint(), what


def rand_values(n, kind, rng):
    if kind == "small":
        return rng.integers(0, 64, n).astype(np.uint64)
    if kind == "wide":
        return rng.integers(0, 2**64 - 1, n, dtype=np.uint64, endpoint=True)
    if kind == "sorted":
        return np.sort(rng.integers(1 << 47, (1 << 47) + 100_000, n)).astype(np.uint64)
    if kind == "runs":
        return np.repeat(rng.integers(0, 5, max(1, n // 7 + 1)), 7)[:n].astype(np.uint64)
    if kind == "outlier":
        x = rng.integers(0, 256, n).astype(np.uint64)
        x[rng.random(n) < 0.01] = rng.integers(0, 1 << 40, int((rng.random(n) < 0.01).sum()) or 1)[0]
        return x
    if kind == "zeros":
        return np.zeros(n, np.uint64)
    raise ValueError(kind)
