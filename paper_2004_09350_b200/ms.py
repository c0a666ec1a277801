"""Python binding of libms (include/ms.h): argument marshalling only.

Every step of every operator runs in libms.so's sm_100a kernels; this module
converts arguments, supplies PyTorch's caching allocator and current CUDA
stream to the library, and owns the returned columns. There is no CPU or
PyTorch fallback: if libms.so is missing, importing this module fails.

Names follow the C ABI (ms_compress -> compress, ...). Citations: PAPER.md
P:n, SPEC.md S:n (see include/ms.h for the per-function contract).
"""
from __future__ import annotations

import ctypes
import os
from typing import NamedTuple, Optional

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libms.so")

UNCOMPR, STATIC_BP, DYN_BP, DELTA_BP, FOR_BP, RLE = range(6)
FORMAT_NAMES = ("UNCOMPR", "STATIC_BP", "DYN_BP", "DELTA_BP", "FOR_BP", "RLE")
EQ, NE, LT, LE, GT, GE, BETWEEN, IN_BITMAP = range(8)
OP_NAMES = ("EQ", "NE", "LT", "LE", "GT", "GE", "BETWEEN", "IN_BITMAP")
STATUS = ("MS_OK", "MS_E_INVALID", "MS_E_WIDTH_OVERFLOW", "MS_E_UNSUPPORTED", "MS_E_RANGE", "MS_E_CORRUPT",
          "MS_E_NOMEM", "MS_E_CUDA")
FLAG_SHRINK = 1
FLAG_GATHER = 2  # ms_project: never stream the data windows (measurement switch)


class MsError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: {STATUS[code] if 0 <= code < len(STATUS) else code}")
        self.code = code


class Fmt(NamedTuple):
    """Column descriptor {format, bit width, block size} (ms_fmt)."""
    format: int
    bit_width: int = 0
    block_size: int = 0

    def __str__(self):
        name = FORMAT_NAMES[self.format]
        if self.format == STATIC_BP:
            return f"{name}{{{self.bit_width or 'auto'}}}"
        if self.format in (DYN_BP, DELTA_BP, FOR_BP):
            return f"{name}{{{self.block_size}}}"
        return name


def uncompr() -> Fmt: return Fmt(UNCOMPR)
def static_bp(w: int = 0) -> Fmt: return Fmt(STATIC_BP, w, 0)
def dyn_bp(B: int = 512) -> Fmt: return Fmt(DYN_BP, 0, B)
def delta_bp(B: int = 512) -> Fmt: return Fmt(DELTA_BP, 0, B)
def for_bp(B: int = 512) -> Fmt: return Fmt(FOR_BP, 0, B)
def rle() -> Fmt: return Fmt(RLE)


class _Fmt(ctypes.Structure):
    _fields_ = [("format", ctypes.c_int32), ("bit_width", ctypes.c_uint32), ("block_size", ctypes.c_uint32),
                ("max_width", ctypes.c_uint32)]


class _Column(ctypes.Structure):
    _fields_ = [("fmt", _Fmt), ("n", ctypes.c_uint64), ("n_blocks", ctypes.c_uint64), ("n_rem", ctypes.c_uint64),
                ("n_runs", ctypes.c_uint64), ("payload_words", ctypes.c_uint64), ("payload", ctypes.c_void_p),
                ("cw", ctypes.c_void_p), ("ref", ctypes.c_void_p), ("rem", ctypes.c_void_p),
                ("alloc", ctypes.c_void_p), ("alloc_bytes", ctypes.c_uint64)]


class _Pred(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("_reserved", ctypes.c_uint32), ("a", ctypes.c_uint64),
                ("b", ctypes.c_uint64), ("bitmap", ctypes.c_void_p), ("bitmap_bits", ctypes.c_uint64)]


_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


class _Ctx(ctypes.Structure):
    _fields_ = [("stream", ctypes.c_void_p), ("alloc", _ALLOC_FN), ("free", _FREE_FN), ("alloc_ctx", ctypes.c_void_p),
                ("flags", ctypes.c_uint32), ("_reserved", ctypes.c_uint32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libms.so not built ({LIB_PATH}); run `python build_native.py libms` — "
                          "there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    C, st, vp, u64 = P(_Column), ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64
    sig = {
        "ms_compress": ([P(_Ctx), vp, u64, _Fmt, C], st),
        "ms_decompress": ([P(_Ctx), C, vp], st),
        "ms_morph": ([P(_Ctx), C, _Fmt, C], st),
        "ms_select": ([P(_Ctx), C, P(_Pred), u64, _Fmt, C], st),
        "ms_project": ([P(_Ctx), C, C, u64, _Fmt, C], st),
        "ms_agg_sum": ([P(_Ctx), C, C, u64, vp], st),
        "ms_agg_sum_grouped": ([P(_Ctx), C, C, u64, vp], st),
        "ms_column_to_device": ([P(_Ctx), C, C], st),
        "ms_column_to_host": ([P(_Ctx), C, C], st),
        "ms_check_errors": ([P(_Ctx)], st),
        "ms_format_sizes": ([P(_Ctx), C, ctypes.c_uint32, vp, P(_Fmt)], st),
        "ms_intersect": ([P(_Ctx), C, C, _Fmt, C], st),
        "ms_merge": ([P(_Ctx), C, C, _Fmt, C], st),
        "ms_group": ([P(_Ctx), C, C, u64, _Fmt, _Fmt, C, C], st),
        "ms_join": ([P(_Ctx), C, C, _Fmt, _Fmt, C, C], st),
        "ms_calc": ([P(_Ctx), ctypes.c_int32, C, C, _Fmt, C], st),
        "ms_semijoin": ([P(_Ctx), C, C, u64, vp, u64, _Fmt, C], st),
        "ms_column_release": ([P(_Ctx), C], None),
        "ms_column_bytes": ([C], u64),
        "ms_status_str": ([ctypes.c_int], ctypes.c_char_p),
        "ms_abi_version": ([], ctypes.c_int),
        "ms_launch_count": ([], u64),
        "ms_profile_enable": ([ctypes.c_int], None),
        "ms_profile_read": ([vp, ctypes.c_int], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    return L


_lib = _load()


def lib():
    return _lib


# ------------------------------------------------------------ allocator
_live = {}


@_ALLOC_FN
def _torch_alloc(_ctx, size, stream):
    try:
        ptr = torch.cuda.caching_allocator_alloc(int(size), torch.cuda.current_device(), int(stream or 0))
        return ptr
    except Exception:  # out of memory -> NULL -> MS_E_NOMEM
        return None


@_FREE_FN
def _torch_free(_ctx, ptr, _stream):
    if ptr:
        torch.cuda.caching_allocator_delete(int(ptr))


_SHIM = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libms_torchalloc.so")
_native_alloc = None


def _alloc_fns():
    """(alloc, free) for ms_ctx: the native shim into PyTorch's caching allocator
    (csrc/shim/torch_alloc.cpp, no Python per allocation) when built, else the
    ctypes callbacks above. Allocation plumbing only; no compute."""
    global _native_alloc
    if _native_alloc is None:
        if os.path.exists(_SHIM):
            shim = ctypes.CDLL(_SHIM)
            _native_alloc = (shim, ctypes.cast(shim.ms_torch_alloc, _ALLOC_FN), ctypes.cast(shim.ms_torch_free, _FREE_FN))
        else:
            _native_alloc = (None, _torch_alloc, _torch_free)
    return _native_alloc[1], _native_alloc[2]


_get_device = torch._C._cuda_getDevice
_get_raw_stream = torch._C._cuda_getCurrentRawStream


def _raw(stream=None) -> int:
    """cudaStream_t of a torch stream, a raw handle, or (None) the current stream —
    without building a torch.cuda.Stream object per call."""
    if stream is None:
        return _get_raw_stream(_get_device())
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


_ctx_cache = {}


def _ctx(stream=None, flags: int = 0) -> _Ctx:
    raw = _raw(stream)
    c = _ctx_cache.get((raw, flags))
    if c is None:
        a, f = _alloc_fns()
        c = _Ctx(stream=raw, alloc=a, free=f, alloc_ctx=None, flags=flags)
        if len(_ctx_cache) < 1024:
            _ctx_cache[(raw, flags)] = c
    return c


def _check(rc: int, where: str):
    if rc != 0:
        raise MsError(rc, where)


def _ptr(t) -> int:
    if isinstance(t, torch.Tensor):
        if not t.is_cuda:
            raise ValueError("device tensor expected")
        if not t.is_contiguous():
            raise ValueError("contiguous tensor expected")
        return t.data_ptr()
    return int(t)


class Column:
    """A device column owned by Python (released through ms_column_release).

    The column's allocation belongs to the stream it was created on (PyTorch's
    caching allocator reuses a freed block in that stream's order). Every op
    records the other streams that read the column; on release the creating
    stream first waits for an event recorded on each of them, so the memory is
    not handed out again while their kernels may still read it."""

    def __init__(self, c: _Column, owned: bool = True, stream=None):
        self._c = c
        self._owned = owned
        self._sraw = _raw(stream)
        self._sobj = stream if isinstance(stream, torch.cuda.Stream) else None
        self._users = None  # raw handle -> torch stream of every other stream that read the column

    def _used_on(self, raw: int, stream):
        if raw != self._sraw:
            if self._users is None:
                self._users = {}
            self._users[raw] = stream if stream is not None else torch.cuda.current_stream()

    def __del__(self):
        try:
            if self._owned and self._c.alloc:
                if self._users:
                    home = self._sobj if self._sobj is not None else torch.cuda.ExternalStream(self._sraw)
                    for s in self._users.values():
                        ev = torch.cuda.Event()
                        ev.record(s)
                        home.wait_event(ev)
                _lib.ms_column_release(ctypes.byref(_ctx(self._sraw)), ctypes.byref(self._c))
        except Exception:
            pass

    @property
    def fmt(self) -> Fmt:
        f = self._c.fmt
        return Fmt(f.format, f.bit_width, f.block_size)

    max_width = property(lambda self: int(self._c.fmt.max_width))  # sizing hint (0 = unknown)
    n = property(lambda self: int(self._c.n))
    n_blocks = property(lambda self: int(self._c.n_blocks))
    n_rem = property(lambda self: int(self._c.n_rem))
    n_runs = property(lambda self: int(self._c.n_runs))
    payload_words = property(lambda self: int(self._c.payload_words))

    def footprint(self) -> int:
        """image bytes: payload + cw + ref + rem (ms_column_bytes)"""
        return int(_lib.ms_column_bytes(ctypes.byref(self._c)))

    def images(self) -> dict:
        """Copy the four image sections to host numpy arrays (ms_column_to_host)."""
        c = self._c
        blockf = c.fmt.format in (DYN_BP, DELTA_BP, FOR_BP)
        out = {
            "payload": np.zeros(c.payload_words, np.uint64),
            "cw": np.zeros(c.n_blocks + 1 if blockf else 0, np.uint32),
            "ref": np.zeros(c.n_blocks if c.fmt.format in (DELTA_BP, FOR_BP) else 0, np.uint64),
            "rem": np.zeros(c.n_rem if blockf else 0, np.uint64),
        }
        h = _Column()
        for k in ("payload", "cw", "ref", "rem"):
            setattr(h, k, out[k].ctypes.data if out[k].size else None)
        _check(_lib.ms_column_to_host(ctypes.byref(_ctx()), ctypes.byref(c), ctypes.byref(h)), "ms_column_to_host")
        return out

    @staticmethod
    def from_host(fmt: Fmt, n: int, payload, cw=None, ref=None, rem=None, n_runs: int = 0) -> "Column":
        """Upload host image sections into a new device column (ms_column_to_device)."""
        h = _Column()
        h.fmt = _Fmt(fmt.format, fmt.bit_width, fmt.block_size, 0)
        h.n = n
        keep = []

        def arr(x, dt):
            a = np.ascontiguousarray(np.asarray(x if x is not None else [], dtype=dt))
            keep.append(a)
            return a

        p = arr(payload, np.uint64)
        h.payload = p.ctypes.data if p.size else None
        h.payload_words = p.size
        if fmt.format in (DYN_BP, DELTA_BP, FOR_BP):
            B = fmt.block_size
            h.n_blocks, h.n_rem = n // B, n % B
            a = arr(cw, np.uint32); h.cw = a.ctypes.data
            a = arr(ref, np.uint64); h.ref = a.ctypes.data if a.size else None
            a = arr(rem, np.uint64); h.rem = a.ctypes.data if a.size else None
        h.n_runs = n_runs
        out = _Column()
        _check(_lib.ms_column_to_device(ctypes.byref(_ctx()), ctypes.byref(h), ctypes.byref(out)),
               "ms_column_to_device")
        torch.cuda.current_stream().synchronize()  # host arrays may be pageable / freed after return
        return Column(out)

    def __repr__(self):
        return f"Column({self.fmt}, n={self.n}, bytes={self.footprint()})"


def _stream_of(stream):
    return stream if stream is not None else _raw(None)


def _uses(stream, *cols):
    """Record that an op on `stream` reads `cols` (see Column); returns the stream
    (its raw handle when None was given)."""
    raw = _raw(stream)
    for c in cols:
        if c is not None:
            c._used_on(raw, stream)
    return stream if stream is not None else raw


def _fmt(f) -> _Fmt:
    f = Fmt(*f) if not isinstance(f, Fmt) else f
    return _Fmt(f.format, f.bit_width, f.block_size, 0)


def compress(values, fmt, n: Optional[int] = None, stream=None, flags: int = 0) -> Column:
    """ms_compress: values = CUDA tensor of 64-bit integers (uint64 bit patterns) or a device pointer."""
    if n is None:
        n = values.numel()
    out = _Column()
    _check(_lib.ms_compress(ctypes.byref(_ctx(stream, flags)), _ptr(values) if n else None, n, _fmt(fmt),
                            ctypes.byref(out)), "ms_compress")
    return Column(out, stream=_stream_of(stream))


def decompress(col: Column, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """ms_decompress into a torch.int64 CUDA tensor (uint64 bit patterns)."""
    if out is None:
        out = torch.empty(col.n, dtype=torch.int64, device="cuda")
    _uses(stream, col)
    _check(_lib.ms_decompress(ctypes.byref(_ctx(stream)), ctypes.byref(col._c), _ptr(out) if col.n else None),
           "ms_decompress")
    return out


def morph(col: Column, fmt, stream=None, flags: int = 0) -> Column:
    out = _Column()
    s = _uses(stream, col)
    _check(_lib.ms_morph(ctypes.byref(_ctx(stream, flags)), ctypes.byref(col._c), _fmt(fmt), ctypes.byref(out)),
           "ms_morph")
    return Column(out, stream=s)


def select(col: Column, op: int, a: int = 0, b: int = 0, bitmap: Optional[torch.Tensor] = None,
           bitmap_bits: int = 0, row_offset: int = 0, out_fmt=None, stream=None, flags: int = 0) -> Column:
    if out_fmt is None:
        out_fmt = delta_bp(512)
    p = _Pred(op=op, a=a & (2**64 - 1), b=b & (2**64 - 1), bitmap=_ptr(bitmap) if bitmap is not None else None,
              bitmap_bits=bitmap_bits)
    out = _Column()
    s = _uses(stream, col)
    _check(_lib.ms_select(ctypes.byref(_ctx(stream, flags)), ctypes.byref(col._c), ctypes.byref(p), row_offset,
                          _fmt(out_fmt), ctypes.byref(out)), "ms_select")
    return Column(out, stream=s)


def project(data: Column, positions: Column, row_offset: int = 0, out_fmt=None, stream=None,
            flags: int = 0) -> Column:
    if out_fmt is None:
        out_fmt = uncompr()
    out = _Column()
    s = _uses(stream, data, positions)
    _check(_lib.ms_project(ctypes.byref(_ctx(stream, flags)), ctypes.byref(data._c), ctypes.byref(positions._c),
                           row_offset, _fmt(out_fmt), ctypes.byref(out)), "ms_project")
    return Column(out, stream=s)


def agg_sum(col: Column, positions: Optional[Column] = None, row_offset: int = 0,
            out: Optional[torch.Tensor] = None, stream=None, check: bool = False) -> torch.Tensor:
    """ms_agg_sum -> 1-element torch.int64 CUDA tensor holding the uint64 sum bits
    (no sync). Device-side errors (a position out of range, a corrupt body) reach
    only the sticky error word: check=True reads it (ms_check_errors, one sync)."""
    if out is None:
        out = torch.empty(1, dtype=torch.int64, device="cuda")
    _uses(stream, col, positions)
    _check(_lib.ms_agg_sum(ctypes.byref(_ctx(stream)), ctypes.byref(col._c),
                           ctypes.byref(positions._c) if positions is not None else None, row_offset, _ptr(out)),
           "ms_agg_sum")
    if check:
        check_errors(stream)
    return out


def agg_sum_grouped(gid: Column, vals: Column, n_groups: int, out: Optional[torch.Tensor] = None,
                    stream=None, check: bool = False) -> torch.Tensor:
    """ms_agg_sum_grouped (no sync); check=True reads the sticky error word (MS_E_RANGE for a gid >= n_groups)."""
    if out is None:
        out = torch.empty(n_groups, dtype=torch.int64, device="cuda")
    _uses(stream, gid, vals)
    _check(_lib.ms_agg_sum_grouped(ctypes.byref(_ctx(stream)), ctypes.byref(gid._c), ctypes.byref(vals._c),
                                   n_groups, _ptr(out) if n_groups else None), "ms_agg_sum_grouped")
    if check:
        check_errors(stream)
    return out


# ------------------------------------------------------------ plan-level operators
CANDIDATES = ("UNCOMPR", "STATIC_BP", "DYN_BP", "DELTA_BP", "FOR_BP", "RLE")  # ms_format_sizes order
ADD, SUB, MUL = 0, 1, 2


def format_sizes(col: Column, block_size: int = 512, stream=None) -> tuple[dict, Fmt]:
    """ms_format_sizes: exact footprint of col in every candidate format (one pass,
    one sync) and the smallest (ties: the simpler format). Returns ({name: bytes}, Fmt)."""
    sizes = np.zeros(6, np.uint64)
    best = _Fmt()
    _uses(stream, col)
    _check(_lib.ms_format_sizes(ctypes.byref(_ctx(stream)), ctypes.byref(col._c), block_size, sizes.ctypes.data,
                                ctypes.byref(best)), "ms_format_sizes")
    return dict(zip(CANDIDATES, (int(x) for x in sizes))), Fmt(best.format, best.bit_width, best.block_size)


def choose_format(col: Column, block_size: int = 512, stream=None) -> Fmt:
    return format_sizes(col, block_size, stream)[1]


def _binary_pos_op(fn, name, a: Column, b: Column, out_fmt, stream):
    out = _Column()
    s = _uses(stream, a, b)
    _check(fn(ctypes.byref(_ctx(stream)), ctypes.byref(a._c), ctypes.byref(b._c), _fmt(out_fmt), ctypes.byref(out)),
           name)
    return Column(out, stream=s)


def intersect(a: Column, b: Column, out_fmt=None, stream=None) -> Column:
    """ms_intersect: sorted intersection of two strictly increasing position columns."""
    return _binary_pos_op(_lib.ms_intersect, "ms_intersect", a, b, out_fmt or delta_bp(512), stream)


def merge(a: Column, b: Column, out_fmt=None, stream=None) -> Column:
    """ms_merge: sorted duplicate-free union of two strictly increasing position columns."""
    return _binary_pos_op(_lib.ms_merge, "ms_merge", a, b, out_fmt or delta_bp(512), stream)


def group(keys: Column, prev_ids: Optional[Column] = None, max_groups: int = 0, ids_fmt=None, extents_fmt=None,
          stream=None) -> tuple[Column, Column]:
    """ms_group -> (group ids, extents)."""
    ids, ext = _Column(), _Column()
    s = _uses(stream, keys, prev_ids)
    _check(_lib.ms_group(ctypes.byref(_ctx(stream)), ctypes.byref(keys._c),
                         ctypes.byref(prev_ids._c) if prev_ids is not None else None, max_groups,
                         _fmt(ids_fmt or uncompr()), _fmt(extents_fmt or uncompr()), ctypes.byref(ids),
                         ctypes.byref(ext)), "ms_group")
    return Column(ids, stream=s), Column(ext, stream=s)


def join(left: Column, right: Column, left_fmt=None, right_fmt=None, stream=None) -> tuple[Column, Column]:
    """ms_join -> (positions into left, positions into right)."""
    lo, ro = _Column(), _Column()
    s = _uses(stream, left, right)
    _check(_lib.ms_join(ctypes.byref(_ctx(stream)), ctypes.byref(left._c), ctypes.byref(right._c),
                        _fmt(left_fmt or uncompr()), _fmt(right_fmt or uncompr()), ctypes.byref(lo),
                        ctypes.byref(ro)), "ms_join")
    return Column(lo, stream=s), Column(ro, stream=s)


def semijoin(keys: Column, positions: Column, bitmap: torch.Tensor, bitmap_bits: int, row_offset: int = 0,
             out_fmt=None, stream=None) -> Column:
    """ms_semijoin: the positions whose key is in the bitmap (fused K7 when the formats allow)."""
    out = _Column()
    s = _uses(stream, keys, positions)
    _check(_lib.ms_semijoin(ctypes.byref(_ctx(stream)), ctypes.byref(keys._c), ctypes.byref(positions._c),
                            row_offset, _ptr(bitmap), bitmap_bits, _fmt(out_fmt or delta_bp(512)),
                            ctypes.byref(out)), "ms_semijoin")
    return Column(out, stream=s)


def calc(op: int, a: Column, b: Column, out_fmt=None, stream=None) -> Column:
    """ms_calc: elementwise ADD / SUB / MUL mod 2^64."""
    out = _Column()
    s = _uses(stream, a, b)
    _check(_lib.ms_calc(ctypes.byref(_ctx(stream)), op, ctypes.byref(a._c), ctypes.byref(b._c),
                        _fmt(out_fmt or uncompr()), ctypes.byref(out)), "ms_calc")
    return Column(out, stream=s)


def check_errors(stream=None):
    _check(_lib.ms_check_errors(ctypes.byref(_ctx(stream))), "ms_check_errors")


def launch_count() -> int:
    return int(_lib.ms_launch_count())


class _KernelTime(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 48), ("launches", ctypes.c_uint64), ("total_ms", ctypes.c_double)]


def profile_enable(on: bool = True):
    """Bracket every libms kernel launch with CUDA events on its stream."""
    _lib.ms_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """{kernel name: (launches, total ms)} since the last read (waits for the events)."""
    buf = (_KernelTime * 64)()
    k = _lib.ms_profile_read(buf, 64)
    return {buf[i].name.decode(): (int(buf[i].launches), float(buf[i].total_ms)) for i in range(min(k, 64))}


def u64(t: torch.Tensor) -> int:
    """uint64 value of a 1-element int64 tensor (bit pattern)."""
    return int(t.item()) & (2**64 - 1)


def to_u64_numpy(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)
