import cProfile, pstats, os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_2004_09350_b200 import ms
n = 1 << 20
X = ms.compress(synth.gen_torch("c5.X", n), ms.dyn_bp(512))
Y = ms.compress(synth.gen_torch("c5.Y", n), ms.for_bp(512))
def run(R):
    for _ in range(R):
        pos = ms.select(X, ms.LT, 1 << 16, out_fmt=ms.delta_bp(512))
        yp = ms.project(Y, pos, 0, ms.for_bp(512))
        s = ms.agg_sum(yp)
    torch.cuda.synchronize()
run(20)
cProfile.run("run(300)", "/tmp/hp.prof")
pstats.Stats("/tmp/hp.prof").sort_stats("tottime").print_stats(25)
