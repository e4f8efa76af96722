"""Launch-list driver for the config-5 and config-4 kernels (run under ncu --metrics gpu__time_duration.sum)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1411_1702_b200 import problems
from paper_1411_1702_b200.sampler import Ensemble, GpuSampler, ObservationModel, PfConfig
n5 = 1 << 25
s = GpuSampler("payload64", PfConfig(particles=n5, seed=5), ObservationModel([0], 1.0))
rng = np.random.default_rng(0)
s.set_ensemble(Ensemble(rng.standard_normal((n5, 6)), rng.standard_normal((n5, 2)), np.zeros(n5), np.zeros(2), np.eye(2)))
s.c5_set_logweights(1.0, 1)
for it in range(3):
    s.c5_iteration(it + 1)
s.synchronize()
s.close()
if "--chain" in sys.argv:
    prob = problems.chain8(particles=1 << 22, T=3, seed=1)
    g = GpuSampler("chain", prob.cfg, prob.obs)
    prob.init(g)
    tp = 0.0
    for j in (1, 2):
        g.pf_step(prob.ys[j - 1], j, tp, prob.times[j - 1], h=prob.h_for(tp, prob.times[j - 1]))
        tp = prob.times[j - 1]
print("ok")
