#!/usr/bin/env python3
"""Kernel times of select X<2^16 -> DELTA_BP{512} on c5-shaped X (DYN_BP{512},
20-bit values) at 2^k rows (libms CUDA-event profiling). For ncu:
-k regex:select_pos. usage: python tools/prof_sel.py [log2 rows ...] [--reps R]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2004_09350_b200 import ms  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    reps = int(os.environ.get("REPS", "5"))
    fmt = os.environ.get("XFMT", "dyn_bp")
    for k in [int(a) for a in args] or [28]:
        n = 1 << k
        X = ms.compress(synth.gen_torch("c5.X", n), ms.dyn_bp(512) if fmt == "dyn_bp" else ms.static_bp(20))
        torch.cuda.synchronize()
        pos = ms.select(X, ms.LT, 1 << 16, out_fmt=ms.delta_bp(512))
        ms.profile_read()
        ms.profile_enable(True)
        for _ in range(reps):
            pos = ms.select(X, ms.LT, 1 << 16, out_fmt=ms.delta_bp(512))
        torch.cuda.synchronize()
        ms.profile_enable(False)
        p = ms.profile_read()
        xb = X.footprint()
        for name, (c, t) in sorted(p.items(), key=lambda kv: -kv[1][1]):
            avg = t / max(c, 1)
            print(f"2^{k}: {name} {avg:.3f} ms  X {xb / 1e9:.3f} GB -> {(xb + pos.footprint()) / avg / 1e6:.0f} GB/s  "
                  f"n_out {pos.n} pos {pos.footprint()} B", flush=True)
        del X, pos
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
