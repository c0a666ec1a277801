python - <<'PY'
import sys; sys.path.insert(0,'.')
import torch, synth
from paper_2004_09350_b200 import ms
n = 1 << 27
x = synth.gen_torch("c3.x", n)
D = ms.compress(x, ms.delta_bp(2048))
R = ms.compress(x, ms.rle())
torch.cuda.synchronize()
m = ms.morph(D, ms.static_bp(0))
u = ms.decompress(D)
v = ms.decompress(R)
torch.cuda.synchronize()
print("ok", m.n)
PY
