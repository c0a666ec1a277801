#!/usr/bin/env python3
"""Build every native artefact of the repo, in-tree (the .so files travel to the
GPU box with the gpurun snapshot).

  synth/libsynth_host.so   gcc   input generators (host)
  synth/libsynth_dev.so    nvcc  input generators (device), sm_100a
  oracle/libms_oracle.so   gcc   the CPU oracle (test infrastructure only)
  paper_2004_09350_b200/libms.so  nvcc  the product: C-ABI library + sm_100a kernels

usage: python build_native.py [synth|oracle|libms|all] [--force]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.check_call(cmd, cwd=ROOT)


def build_synth(force=False):
    d = os.path.join(ROOT, "synth")
    hdr = os.path.join(d, "synth.h")
    host_src = os.path.join(d, "synth_host.c")
    host_so = os.path.join(d, "libsynth_host.so")
    if force or _stale(host_so, [host_src, hdr]):
        _run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", host_so, host_src])
    dev_src = os.path.join(d, "synth_dev.cu")
    dev_so = os.path.join(d, "libsynth_dev.so")
    if force or _stale(dev_so, [dev_src, hdr]):
        _run([NVCC, *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-o", dev_so, dev_src])


def build_oracle(force=False):
    d = os.path.join(ROOT, "oracle")
    srcs = sorted(glob.glob(os.path.join(d, "*.c")))
    hdrs = sorted(glob.glob(os.path.join(d, "*.h"))) + [os.path.join(ROOT, "synth", "synth.h")]
    so = os.path.join(d, "libms_oracle.so")
    if srcs and (force or _stale(so, srcs + hdrs)):
        _run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-I", os.path.join(ROOT, "synth"),
              "-o", so, *srcs])


def _local_deps(path, dirs, seen=None):
    """The file plus every quoted #include it pulls in (recursively) from dirs."""
    import re
    seen = set() if seen is None else seen
    if path in seen:
        return seen
    seen.add(path)
    for inc in re.findall(r'^\s*#\s*include\s+"([^"]+)"', open(path).read(), re.M):
        for d in dirs:
            q = os.path.join(d, inc)
            if os.path.exists(q):
                _local_deps(q, dirs, seen)
                break
    return seen


def build_libms(force=False):
    from concurrent.futures import ThreadPoolExecutor
    pkg = os.path.join(ROOT, "paper_2004_09350_b200")
    csrc = os.path.join(pkg, "csrc")
    inc = os.path.join(ROOT, "include")
    srcs = sorted(glob.glob(os.path.join(csrc, "*.cu")))
    so = os.path.join(pkg, "libms.so")
    objdir = os.path.join(ROOT, "build", "libms")
    os.makedirs(objdir, exist_ok=True)
    flags = [*ARCH, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler",
             "-fvisibility=hidden", "-I", inc, "-I", csrc,
             "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
    objs, jobs = [], []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        if force or _stale(o, sorted(_local_deps(s, [csrc, inc]))):
            jobs.append([NVCC, *flags, "-c", "-o", o, s])
        objs.append(o)
    if jobs:
        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1)) as ex:
            list(ex.map(_run, jobs))
    stale_objs = [o for o in glob.glob(os.path.join(objdir, "*.o")) if o not in objs]
    for o in stale_objs:  # objects of sources that no longer exist
        os.unlink(o)
    if force or jobs or _stale(so, objs):
        _run([NVCC, *ARCH, "-shared", "-o", so, *objs, "-lcudart"])


def build_shim(force=False):
    """paper_2004_09350_b200/libms_torchalloc.so: ms_ctx alloc/free callbacks into
    PyTorch's CUDA caching allocator (g++, torch headers; plumbing, no compute)."""
    import sysconfig  # noqa: F401
    try:
        import torch
    except Exception:  # torch missing: the binding falls back to ctypes callbacks
        return
    pkg = os.path.join(ROOT, "paper_2004_09350_b200")
    src = os.path.join(pkg, "csrc", "shim", "torch_alloc.cpp")
    so = os.path.join(pkg, "libms_torchalloc.so")
    if not (force or _stale(so, [src])):
        return
    tdir = os.path.dirname(torch.__file__)
    abi = int(torch._C._GLIBCXX_USE_CXX11_ABI)
    _run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", f"-D_GLIBCXX_USE_CXX11_ABI={abi}",
          "-I", os.path.join(tdir, "include"), "-I", "/usr/local/cuda/include", src, "-o", so,
          "-L", os.path.join(tdir, "lib"), "-lc10", "-lc10_cuda", "-Wl,-rpath," + os.path.join(tdir, "lib")])


def build_all(force=False):
    build_synth(force)
    build_oracle(force)
    build_libms(force)
    build_shim(force)


if __name__ == "__main__":
    what = [a for a in sys.argv[1:] if not a.startswith("--")] or ["all"]
    force = "--force" in sys.argv
    for w in what:
        {"synth": build_synth, "oracle": build_oracle, "libms": build_libms, "shim": build_shim,
         "all": build_all}[w](force)
