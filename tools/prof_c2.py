import sys, torch
sys.path.insert(0, '/root/repo')
import synth
from paper_2004_09350_b200 import ms
n = 1 << 28
X = ms.compress(synth.gen_torch("c2.X", n), ms.dyn_bp(512))
print("X bytes", X.footprint(), "maxw", X.max_width)
ms.select(X, ms.EQ, 17, out_fmt=ms.delta_bp(512)); torch.cuda.synchronize()
ms.profile_read(); ms.profile_enable(True)
for _ in range(5): ms.select(X, ms.EQ, 17, out_fmt=ms.delta_bp(512))
torch.cuda.synchronize(); ms.profile_enable(False)
for k, (c, t) in sorted(ms.profile_read().items(), key=lambda kv: -kv[1][1]): print(k, round(t / c, 4))
