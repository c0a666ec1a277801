python - <<'PY'
import sys; sys.path.insert(0,'.')
import torch, synth
from paper_2004_09350_b200 import ms
n = 1 << 27
x = synth.gen_torch("c2.X", n)
D = ms.compress(x, ms.dyn_bp(512))
torch.cuda.synchronize()
D = ms.compress(x, ms.dyn_bp(512))
torch.cuda.synchronize()
print("ok", D.n)
PY
