"""Where the literal Ensemble& drop-in step spends its time (LV 2^20)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_1702_b200 import problems  # noqa: E402
from paper_1411_1702_b200.sampler import GpuSampler  # noqa: E402

n = 1 << 20
prob = problems.lotka_volterra(particles=n, T=30, seed=1)
g = GpuSampler("lv", prob.cfg, prob.obs)
g.initialize_uniform(**prob.prior)
ens = g.get_ensemble()
tp = 0.0
for j in range(1, 8):
    t0 = time.perf_counter()
    g.set_ensemble(ens)
    t1 = time.perf_counter()
    g.pf_step(prob.ys[j - 1], j, tp, prob.times[j - 1])
    t2 = time.perf_counter()
    ens = g.get_ensemble()
    t3 = time.perf_counter()
    tp = prob.times[j - 1]
    print(f"set {1e3 * (t1 - t0):.2f} ms  step {1e3 * (t2 - t1):.2f} ms  get {1e3 * (t3 - t2):.2f} ms")
