"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Thin ctypes wrapper over oracle/libms_oracle.so (plain C, see ms_oracle.h).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package; the product path never does.

Columns are returned as `OColumn`: numpy copies of the four image sections
(payload, cw, ref, rem) plus the descriptor fields, so tests can compare the
GPU image section by section (SURVEY.md §8(c) c.2 "image").
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "libms_oracle.so")

UNCOMPR, STATIC_BP, DYN_BP, DELTA_BP, FOR_BP, RLE = range(6)
FORMAT_NAMES = {UNCOMPR: "UNCOMPR", STATIC_BP: "STATIC_BP", DYN_BP: "DYN_BP", DELTA_BP: "DELTA_BP",
                FOR_BP: "FOR_BP", RLE: "RLE"}
EQ, NE, LT, LE, GT, GE, BETWEEN, IN_BITMAP = range(8)
OK, E_INVALID, E_WIDTH_OVERFLOW, E_UNSUPPORTED, E_RANGE, E_CORRUPT, E_NOMEM = range(7)


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle status {code}")
        self.code = code


class _Col(ctypes.Structure):
    _fields_ = [
        ("format", ctypes.c_int32), ("bit_width", ctypes.c_uint32), ("block_size", ctypes.c_uint32),
        ("_pad", ctypes.c_uint32),
        ("n", ctypes.c_uint64), ("n_blocks", ctypes.c_uint64), ("n_rem", ctypes.c_uint64),
        ("n_runs", ctypes.c_uint64), ("payload_words", ctypes.c_uint64),
        ("payload", ctypes.POINTER(ctypes.c_uint64)), ("cw", ctypes.POINTER(ctypes.c_uint32)),
        ("ref", ctypes.POINTER(ctypes.c_uint64)), ("rem", ctypes.POINTER(ctypes.c_uint64)),
    ]


@dataclass
class OColumn:
    format: int
    bit_width: int
    block_size: int
    n: int
    n_blocks: int
    n_rem: int
    n_runs: int
    payload: np.ndarray
    cw: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    ref: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    rem: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))

    @property
    def payload_words(self):
        return int(self.payload.size)

    def footprint(self) -> int:
        b = 8 * self.payload.size
        if self.format in (DYN_BP, DELTA_BP, FOR_BP):
            b += 4 * (self.n_blocks + 1) + 8 * self.n_rem
            if self.format != DYN_BP:
                b += 8 * self.n_blocks
        return int(b)

    def _c(self) -> _Col:
        # keep contiguous arrays alive on self while the struct is in use
        self._keep = [np.ascontiguousarray(self.payload, np.uint64),
                      np.ascontiguousarray(self.cw, np.uint32),
                      np.ascontiguousarray(self.ref, np.uint64),
                      np.ascontiguousarray(self.rem, np.uint64)]
        p, cw, ref, rem = self._keep
        c = _Col(format=self.format, bit_width=self.bit_width, block_size=self.block_size,
                 n=self.n, n_blocks=self.n_blocks, n_rem=self.n_rem, n_runs=self.n_runs,
                 payload_words=p.size)
        c.payload = p.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
        c.cw = cw.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
        c.ref = ref.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
        c.rem = rem.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
        return c


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} missing: run `python build_native.py oracle`")
        L = ctypes.CDLL(LIB)
        P = ctypes.POINTER
        u64, u32, i32, vp = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int32, ctypes.c_void_p
        L.orc_ebw.argtypes = [u64]; L.orc_ebw.restype = u32
        L.orc_pack.argtypes = [vp, u64, u32, vp]; L.orc_pack.restype = ctypes.c_int
        L.orc_unpack.argtypes = [vp, u64, u32, vp]; L.orc_unpack.restype = None
        L.orc_get_at.argtypes = [vp, u32, u64]; L.orc_get_at.restype = u64
        L.orc_encode.argtypes = [vp, u64, i32, u32, u32, P(_Col)]; L.orc_encode.restype = ctypes.c_int
        L.orc_decode.argtypes = [P(_Col), vp]; L.orc_decode.restype = ctypes.c_int
        L.orc_free.argtypes = [P(_Col)]; L.orc_free.restype = None
        L.orc_footprint.argtypes = [P(_Col)]; L.orc_footprint.restype = u64
        L.orc_select.argtypes = [P(_Col), i32, u64, u64, vp, u64, u64, i32, u32, u32, P(_Col)]
        L.orc_select.restype = ctypes.c_int
        L.orc_project.argtypes = [P(_Col), P(_Col), u64, i32, u32, u32, P(_Col)]
        L.orc_project.restype = ctypes.c_int
        L.orc_agg_sum.argtypes = [P(_Col), P(_Col), u64, P(u64)]; L.orc_agg_sum.restype = ctypes.c_int
        L.orc_agg_sum_grouped.argtypes = [P(_Col), P(_Col), u64, vp]
        L.orc_agg_sum_grouped.restype = ctypes.c_int
        L.orc_morph.argtypes = [P(_Col), i32, u32, u32, P(_Col)]; L.orc_morph.restype = ctypes.c_int
        L.orc_count_raw.argtypes = [vp, u64, i32, u64, u64, vp, u64]; L.orc_count_raw.restype = u64
        _lib = L
    return _lib


def _check(rc):
    if rc != OK:
        raise OracleError(rc)


def _take(c: _Col) -> OColumn:
    """Copy a C-owned column into numpy arrays and free the C side."""
    def arr(ptr, n, dt):
        if n == 0 or not ptr:
            return np.zeros(0, dt)
        return np.ctypeslib.as_array(ptr, shape=(n,)).copy()
    blockf = c.format in (DYN_BP, DELTA_BP, FOR_BP)
    oc = OColumn(format=c.format, bit_width=c.bit_width, block_size=c.block_size, n=c.n,
                 n_blocks=c.n_blocks, n_rem=c.n_rem, n_runs=c.n_runs,
                 payload=arr(c.payload, c.payload_words, np.uint64),
                 cw=arr(c.cw, c.n_blocks + 1, np.uint32) if blockf else np.zeros(0, np.uint32),
                 ref=arr(c.ref, c.n_blocks, np.uint64) if c.format in (DELTA_BP, FOR_BP)
                 else np.zeros(0, np.uint64),
                 rem=arr(c.rem, c.n_rem, np.uint64) if blockf else np.zeros(0, np.uint64))
    lib().orc_free(ctypes.byref(c))
    return oc


def _u64(v) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.uint64))


def ebw(v: int) -> int:
    return int(lib().orc_ebw(int(v)))


def pack(values, w: int) -> np.ndarray:
    v = _u64(values)
    out = np.zeros((v.size * w + 63) // 64, np.uint64)
    _check(lib().orc_pack(v.ctypes.data, v.size, w, out.ctypes.data))
    return out


def unpack(words, n: int, w: int) -> np.ndarray:
    wd = _u64(words)
    out = np.zeros(n, np.uint64)
    lib().orc_unpack(wd.ctypes.data, n, w, out.ctypes.data)
    return out


def get_at(words, w: int, i: int) -> int:
    wd = _u64(words)
    return int(lib().orc_get_at(wd.ctypes.data, w, i))


def encode(values, fmt: int, bit_width: int = 0, block_size: int = 0) -> OColumn:
    v = _u64(values)
    c = _Col()
    _check(lib().orc_encode(v.ctypes.data, v.size, fmt, bit_width, block_size, ctypes.byref(c)))
    return _take(c)


def decode(col: OColumn) -> np.ndarray:
    out = np.zeros(col.n, np.uint64)
    c = col._c()
    _check(lib().orc_decode(ctypes.byref(c), out.ctypes.data))
    return out


def select(col: OColumn, op: int, a: int = 0, b: int = 0, bitmap=None, bitmap_bits: int = 0,
           row_offset: int = 0, out_fmt: int = DELTA_BP, out_width: int = 0, out_block: int = 512):
    bm = _u64(bitmap) if bitmap is not None else np.zeros(1, np.uint64)
    c = col._c()
    o = _Col()
    _check(lib().orc_select(ctypes.byref(c), op, a, b, bm.ctypes.data, bitmap_bits, row_offset,
                            out_fmt, out_width, out_block, ctypes.byref(o)))
    return _take(o)


def project(data: OColumn, pos: OColumn, row_offset: int = 0, out_fmt: int = UNCOMPR,
            out_width: int = 0, out_block: int = 512) -> OColumn:
    d, p = data._c(), pos._c()
    o = _Col()
    _check(lib().orc_project(ctypes.byref(d), ctypes.byref(p), row_offset, out_fmt, out_width, out_block,
                             ctypes.byref(o)))
    return _take(o)


def agg_sum(col: OColumn, pos: OColumn | None = None, row_offset: int = 0) -> int:
    c = col._c()
    s = ctypes.c_uint64(0)
    if pos is None:
        _check(lib().orc_agg_sum(ctypes.byref(c), None, row_offset, ctypes.byref(s)))
    else:
        p = pos._c()
        _check(lib().orc_agg_sum(ctypes.byref(c), ctypes.byref(p), row_offset, ctypes.byref(s)))
    return int(s.value)


def agg_sum_grouped(gid: OColumn, vals: OColumn, n_groups: int) -> np.ndarray:
    g, v = gid._c(), vals._c()
    out = np.zeros(n_groups, np.uint64)
    _check(lib().orc_agg_sum_grouped(ctypes.byref(g), ctypes.byref(v), n_groups, out.ctypes.data))
    return out


def morph(col: OColumn, fmt: int, bit_width: int = 0, block_size: int = 0) -> OColumn:
    c = col._c()
    o = _Col()
    _check(lib().orc_morph(ctypes.byref(c), fmt, bit_width, block_size, ctypes.byref(o)))
    return _take(o)


def count_raw(values, op: int, a: int = 0, b: int = 0, bitmap=None, bitmap_bits: int = 0) -> int:
    v = _u64(values)
    bm = _u64(bitmap) if bitmap is not None else np.zeros(1, np.uint64)
    return int(lib().orc_count_raw(v.ctypes.data, v.size, op, a, b, bm.ctypes.data, bitmap_bits))
