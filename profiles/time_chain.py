"""ms per chain (BASELINE config 4) step at 2^22 (quick A/B timing)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1411_1702_b200 import problems
from paper_1411_1702_b200.sampler import GpuSampler
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
prob = problems.chain8(particles=n, T=8, seed=1)
g = GpuSampler("chain", prob.cfg, prob.obs)
prob.init(g)
tp, ms = 0.0, []
for j in range(1, 7):
    t1 = prob.times[j - 1]
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g.pf_step(prob.ys[j - 1], j, tp, t1, h=prob.h_for(tp, t1))
    torch.cuda.synchronize(); ms.append(1e3 * (time.perf_counter() - t0))
    tp = t1
print("chain ms/step", [round(x, 2) for x in ms], "mean(last 4)", round(sum(ms[2:]) / 4, 3))
