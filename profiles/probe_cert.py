"""Uncertain-slot counts of the certified CDF per LV step (2^20 default)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_1702_b200 import problems  # noqa: E402
from paper_1411_1702_b200.sampler import GpuSampler  # noqa: E402

n = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 20)
prob = problems.lotka_volterra(particles=n, T=30, seed=1)
g = GpuSampler("lv", prob.cfg, prob.obs)
g.initialize_uniform(**prob.prior)
tp = 0.0
out = []
for j in range(1, 21):
    g.pf_step(prob.ys[j - 1], j, tp, prob.times[j - 1])
    tp = prob.times[j - 1]
    out.append(g.uncertain_slots())
print("uncertain per step:", out)
