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


def build_libms(force=False):
    pkg = os.path.join(ROOT, "paper_2004_09350_b200")
    csrc = os.path.join(pkg, "csrc")
    srcs = sorted(glob.glob(os.path.join(csrc, "*.cu")))
    hdrs = sorted(glob.glob(os.path.join(csrc, "*.cuh"))) + sorted(
        glob.glob(os.path.join(ROOT, "include", "*.h")))
    so = os.path.join(pkg, "libms.so")
    if not srcs or not (force or _stale(so, srcs + hdrs)):
        return
    objdir = os.path.join(ROOT, "build", "libms")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    flags = [*ARCH, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler",
             "-fvisibility=hidden", "-I", os.path.join(ROOT, "include"), "-I", csrc,
             "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        if force or _stale(o, [s] + hdrs):
            _run([NVCC, *flags, "-c", "-o", o, s])
        objs.append(o)
    _run([NVCC, *ARCH, "-shared", "-o", so, *objs, "-lcudart"])


def build_all(force=False):
    build_synth(force)
    build_oracle(force)
    build_libms(force)


if __name__ == "__main__":
    what = [a for a in sys.argv[1:] if not a.startswith("--")] or ["all"]
    force = "--force" in sys.argv
    for w in what:
        {"synth": build_synth, "oracle": build_oracle, "libms": build_libms, "all": build_all}[w](force)
