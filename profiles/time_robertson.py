"""ms per Robertson (BASELINE config 3) step at 2^22 (quick A/B timing)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1411_1702_b200 import problems
from paper_1411_1702_b200.sampler import GpuSampler
n = 1 << 22
prob = problems.robertson(particles=n, T=400, seed=1)
g = GpuSampler("robertson", prob.cfg, prob.obs)
prob.init(g)
tp, ms = 0.0, []
for j in range(1, 9):
    t1 = prob.times[j - 1]
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g.pf_step(prob.ys[j - 1], j, tp, t1, h=prob.h_for(tp, t1))
    torch.cuda.synchronize(); ms.append(1e3 * (time.perf_counter() - t0))
    tp = t1
print("robertson ms/step mean(last 6)", round(sum(ms[2:]) / 6, 3))
