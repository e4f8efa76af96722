"""Runs a few steps of a stiff BASELINE workload for ncu captures.

  python profiles/probe_stiff.py chain|robertson exact|fast [n_log2]
Robertson is advanced to the stiff part of the grid (j = 200) first.
"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_1702_b200 import problems  # noqa: E402
from paper_1411_1702_b200.sampler import GpuSampler  # noqa: E402

model, arith = sys.argv[1], sys.argv[2]
n = 1 << int(sys.argv[3]) if len(sys.argv) > 3 else (1 << 22)
prob = problems.chain8(particles=n, T=10, seed=1) if model == "chain" else problems.robertson(particles=n, T=400, seed=1)
g = GpuSampler(model, dataclasses.replace(prob.cfg, arithmetic=arith), prob.obs)
prob.init(g)
j0 = 0 if model == "chain" else 199
tp = 0.0
for j in range(1, j0 + 4):
    t1 = prob.times[j - 1]
    g.pf_step(prob.ys[j - 1], j, tp, t1, h=prob.h_for(tp, t1))
    tp = t1
g.synchronize()
print("done", model, arith, n)
