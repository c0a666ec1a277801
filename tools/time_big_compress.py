#!/usr/bin/env python3
"""Wall time of compressing the full c5 column (2^32 rows) to DYN_BP / FOR_BP (bench setup size)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2004_09350_b200 import ms  # noqa: E402

torch.cuda.set_device(0)
n = 1 << 32
x = synth.gen_torch("c5.X", n)
for f, name in ((ms.dyn_bp(512), "DYN_BP{512}"), (ms.for_bp(512), "FOR_BP{512}")):
    torch.cuda.synchronize(); t = time.time(); X = ms.compress(x, f); torch.cuda.synchronize()
    print(name, "first", round((time.time() - t) * 1e3, 1), "ms")
    torch.cuda.synchronize(); t = time.time(); X = ms.compress(x, f); torch.cuda.synchronize()
    print(name, "second", round((time.time() - t) * 1e3, 1), "ms", X.footprint())
    del X
