"""Seeded synthetic inputs shared by the oracle side and the GPU side.

Input generation only (no formats, no operators): see synth.h for the exact
definitions. The recipes below restate SURVEY.md §8(d) d.2 / d.2b, which give
BASELINE.json's five configs and the paper's Table `tab:datach` columns
 a concrete, counter-based definition. Every input in the
tests and in bench.py comes from here; nothing is read from disk.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
HOST_LIB = os.path.join(_HERE, "libsynth_host.so")
DEV_LIB = os.path.join(_HERE, "libsynth_dev.so")

SYN_MASK, SYN_RANGE, SYN_OUTLIER, SYN_RUNS = 0, 1, 2, 3
M64 = (1 << 64) - 1


class Recipe(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_uint32), ("skew", ctypes.c_uint32),
        ("seed", ctypes.c_uint64), ("seed2", ctypes.c_uint64),
        ("mask", ctypes.c_uint64), ("mask2", ctypes.c_uint64),
        ("m", ctypes.c_uint64), ("add", ctypes.c_uint64),
        ("outlier_const", ctypes.c_uint64),
        ("skew_seed", ctypes.c_uint64), ("skew_low", ctypes.c_uint64), ("skew_m", ctypes.c_uint64),
    ]


def mix64(z: int) -> int:
    z &= M64
    z ^= z >> 30; z = (z * 0xBF58476D1CE4E5B9) & M64
    z ^= z >> 27; z = (z * 0x94D049BB133111EB) & M64
    z ^= z >> 31
    return z


def seed(c: int) -> int:
    """Stream seed s_c: s_0 = 42, s_c = mix64(42 + c)."""
    return 42 if c == 0 else mix64(42 + c)


def recipe(kind, seed=0, seed2=0, mask=0, mask2=0, m=0, add=0, outlier_const=0,
           skew=None, sorted_=False):
    r = Recipe(kind=kind, skew=0, seed=seed, seed2=seed2, mask=mask, mask2=mask2, m=m,
               add=add, outlier_const=outlier_const)
    if skew is not None:
        r.skew = 1
        r.skew_seed, r.skew_low, r.skew_m = skew
    r.sorted_ = sorted_  # python-side attribute: host sorts after generation (pin C4 only)
    return r


D4 = (2556, 200_000, 3_000_000, 130_000)

RECIPES = {
    # BASELINE.json configs[0..4]
    "c1.X": lambda: recipe(SYN_MASK, seed=seed(0), mask=1023),
    "c2.X": lambda: recipe(SYN_OUTLIER, seed=seed(1), seed2=seed(2), m=100, mask=255,
                           mask2=(1 << 40) - 1),
    "c2.Y": lambda: recipe(SYN_MASK, seed=seed(3), mask=(1 << 20) - 1, add=10**6),
    "c3.x": lambda: recipe(SYN_RUNS, seed=seed(4)),
    "c4.k0": lambda: recipe(SYN_RANGE, seed=seed(5), m=D4[0]),
    "c4.k1": lambda: recipe(SYN_RANGE, seed=seed(6), m=D4[1]),
    "c4.k2": lambda: recipe(SYN_RANGE, seed=seed(7), m=D4[2]),
    "c4.k3": lambda: recipe(SYN_RANGE, seed=seed(8), m=D4[3]),
    "c4.m1": lambda: recipe(SYN_RANGE, seed=seed(9), m=10**5, add=1),
    "c4.m2": lambda: recipe(SYN_RANGE, seed=seed(10), m=10**5, add=1),
    "c4.bitmapU": lambda: recipe(SYN_RANGE, seed=seed(11), m=25),   # bit k set <=> value == 0
    "c4.gattr": lambda: recipe(SYN_RANGE, seed=seed(12), m=1000),
    "c5.X": lambda: recipe(SYN_MASK, seed=seed(13), mask=(1 << 20) - 1),
    "c5.Y": lambda: recipe(SYN_MASK, seed=seed(14), mask=(1 << 20) - 1, add=10**6),
    # the paper's synthetic columns, Table tab:datach;
    # X carries the select benchmark's 90% lowest-value skew
    "C1.X": lambda: recipe(SYN_MASK, seed=seed(21), mask=63, skew=(seed(20), 0, 10)),
    "C1.Y": lambda: recipe(SYN_MASK, seed=seed(22), mask=63),
    "C1.plain": lambda: recipe(SYN_MASK, seed=seed(21), mask=63),
    "C2.X": lambda: recipe(SYN_OUTLIER, seed=seed(23), seed2=seed(24), m=10000, mask=63,
                           mask2=(1 << 63) - 1, outlier_const=1, skew=(seed(20), 0, 10)),
    "C2.plain": lambda: recipe(SYN_OUTLIER, seed=seed(23), seed2=seed(24), m=10000, mask=63,
                               mask2=(1 << 63) - 1, outlier_const=1),
    "C3.X": lambda: recipe(SYN_MASK, seed=seed(21), mask=63, add=1 << 62,
                           skew=(seed(20), 1 << 62, 10)),
    "C3.Y": lambda: recipe(SYN_MASK, seed=seed(22), mask=63, add=1 << 62),
    "C4.Y": lambda: recipe(SYN_RANGE, seed=seed(22), m=100_001, add=1 << 47, sorted_=True),
    # C4 with the select benchmark's 90% lowest-value skew, then sorted
    "C4.X": lambda: recipe(SYN_RANGE, seed=seed(22), m=100_001, add=1 << 47, sorted_=True,
                           skew=(seed(20), 1 << 47, 10)),
}

_host = None
_dev = None


def _host_lib():
    global _host
    if _host is None:
        if not os.path.exists(HOST_LIB):
            raise RuntimeError(f"{HOST_LIB} missing: run `python build_native.py synth`")
        _host = ctypes.CDLL(HOST_LIB)
        _host.synth_fill_host.argtypes = [ctypes.POINTER(Recipe), ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.c_void_p]
        _host.synth_fill_host.restype = None
    return _host


def _dev_lib():
    global _dev
    if _dev is None:
        if not os.path.exists(DEV_LIB):
            raise RuntimeError(f"{DEV_LIB} missing: run `python build_native.py synth`")
        _dev = ctypes.CDLL(DEV_LIB)
        _dev.synth_fill_device.argtypes = [ctypes.POINTER(Recipe), ctypes.c_uint64, ctypes.c_uint64,
                                           ctypes.c_void_p, ctypes.c_void_p]
        _dev.synth_fill_device.restype = ctypes.c_int
    return _dev


def get(name_or_recipe) -> Recipe:
    if isinstance(name_or_recipe, Recipe):
        return name_or_recipe
    return RECIPES[name_or_recipe]()


def gen_host(name_or_recipe, n: int, start: int = 0) -> np.ndarray:
    """Rows [start, start+n) of a recipe as a uint64 numpy array (host C)."""
    r = get(name_or_recipe)
    out = np.empty(int(n), dtype=np.uint64)
    if n:
        _host_lib().synth_fill_host(ctypes.byref(r), start, n, out.ctypes.data)
    if getattr(r, "sorted_", False):
        out.sort()
    return out


def gen_device(name_or_recipe, n: int, out_ptr: int, stream_ptr: int = 0, start: int = 0) -> None:
    """Rows [start, start+n) of a recipe into a device buffer (CUDA, own library)."""
    r = get(name_or_recipe)
    if getattr(r, "sorted_", False):
        raise ValueError("sorted recipes are host-only")
    rc = _dev_lib().synth_fill_device(ctypes.byref(r), start, n, out_ptr, stream_ptr)
    if rc != 0:
        raise RuntimeError(f"synth_fill_device failed: cuda error {rc}")


def gen_torch(name_or_recipe, n: int, device="cuda", start: int = 0):
    """Convenience: a torch.int64 CUDA tensor holding the uint64 bit patterns."""
    import torch
    t = torch.empty(int(n), dtype=torch.int64, device=device)
    if n:
        gen_device(name_or_recipe, n, t.data_ptr(), torch.cuda.current_stream(t.device).cuda_stream,
                   start)
    return t


def bitmap_c4() -> np.ndarray:
    """c4 dimension bitmap over the k1 domain: bit k set <=> U(R(s11,k),25) == 0 (D-16)."""
    u = gen_host("c4.bitmapU", D4[1])
    bits = (u == 0)
    words = np.zeros((D4[1] + 63) // 64, dtype=np.uint64)
    idx = np.nonzero(bits)[0]
    np.bitwise_or.at(words, idx // 64, (np.uint64(1) << (idx % 64).astype(np.uint64)))
    return words
