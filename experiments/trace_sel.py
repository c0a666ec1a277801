#!/usr/bin/env python3
"""Per-tile phase timeline of the one-pass select (ms_debug_trace): c5-shaped X
at 2^k rows, select X < 2^16 -> DELTA_BP{512}; prints per-phase duration
percentiles and the spread of tile completions.
usage: python tools/trace_sel.py [log2 rows]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2004_09350_b200 import ms  # noqa: E402

PH = ["mask", "enc_start", "tail", "lb1", "head", "pass1", "lb2", "stored"]


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    n = 1 << k
    X = ms.compress(synth.gen_torch("c5.X", n), ms.dyn_bp(512))
    T = int(ms.lib().ms_debug_trace_tiles(n))
    buf = torch.zeros(T * 16, dtype=torch.int64, device="cuda")
    ms.select(X, ms.LT, 1 << 16, out_fmt=ms.delta_bp(512))
    torch.cuda.synchronize()
    assert ms.lib().ms_debug_trace(buf.data_ptr()) == 0
    ms.select(X, ms.LT, 1 << 16, out_fmt=ms.delta_bp(512))
    torch.cuda.synchronize()
    ms.lib().ms_debug_trace(None)
    full = buf.cpu().numpy().reshape(T, 16).astype(np.int64)
    tr = full[:, :8]
    ctr = full[:, 8:]
    for k, name in ((0, "locate+scan cyc"), (1, "scatter cyc"), (2, "fill cyc"), (3, "deltas cyc"),
                    (4, "warp1 pass1 total cyc"), (5, "span words"), (6, "blocks/tile")):
        v = ctr[:, k][ctr[:, k] > 0]
        if v.size:
            print(f"{name:>22}: p50 {np.percentile(v, 50):9.0f}  p90 {np.percentile(v, 90):9.0f}")
    t0 = tr[tr > 0].min()
    tr = np.where(tr > 0, tr - t0, -1)
    print(f"2^{k} rows, {T} tiles, span {tr.max() / 1e3:.1f} us")
    for i in range(1, 8):
        d = tr[:, i] - tr[:, i - 1]
        d = d[(tr[:, i] >= 0) & (tr[:, i - 1] >= 0)]
        if d.size:
            print(f"{PH[i - 1]:>9} -> {PH[i]:<9} p10 {np.percentile(d, 10) / 1e3:7.2f}  p50 {np.percentile(d, 50) / 1e3:7.2f}"
                  f"  p90 {np.percentile(d, 90) / 1e3:7.2f}  max {d.max() / 1e3:7.2f} us")
    m = tr[:, 0]
    print("mask-complete times (us) of tiles 0..9:", (m[:10] / 1e3).round(2).tolist())
    print("stored times (us) of tiles 0..9:", (tr[:10, 7] / 1e3).round(2).tolist())
    gaps = np.diff(np.sort(m)) / 1e3
    print(f"mask completions: mean gap {gaps.mean():.3f} us; per CTA period ~ {gaps.mean() * 148:.2f} us")


if __name__ == "__main__":
    main()
