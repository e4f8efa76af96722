"""A few chain (BASELINE config 4) steps at 2^22 for profiling."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_1702_b200 import problems
from paper_1411_1702_b200.sampler import GpuSampler
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
prob = problems.chain8(particles=n, T=4, seed=1)
g = GpuSampler("chain", prob.cfg, prob.obs)
prob.init(g)
tp = 0.0
for j in (1, 2, 3):
    g.pf_step(prob.ys[j - 1], j, tp, prob.times[j - 1], h=prob.h_for(tp, prob.times[j - 1]))
    tp = prob.times[j - 1]
print("ok")
