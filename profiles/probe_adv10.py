"""Timing probe: the advdiff kernels at n = 10 (m = 9), 5000 particles, BDF2 h = 0.05."""
import json, sys, os
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_1411_1702_b200 import problems
from paper_1411_1702_b200.sampler import GpuSampler
prob = problems.advdiff(particles=5000, n=10, seed=1)
prob.obs.sigma *= 10.0  # a timing probe: keep the posterior from collapsing (chol_psd) within the steps
g = GpuSampler("advdiff", prob.cfg, prob.obs, model_consts=prob.model_consts)
prob.init(g)
ms, it = bench._timed_steps(g, prob, 2, 1, torch.cuda.ExternalStream(g.stream_handle))
print(json.dumps({"ms": sum(ms) / len(ms)}))
