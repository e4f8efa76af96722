"""A/B timing of two library builds on BASELINE config 4 (chain, BDF3 m = 3)
or the reference's problem 1 (metabolic, BDF2 m = 4):
    python profiles/ab_chain.py A.so B.so [rounds] [n] [chain|metabolic|robertson|lv] [exact|fast]
Each run: a fresh process, 2 warm-up + 3 timed drop-in steps at n particles
(device events), alternating builds; prints ms/step and the medians."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import dataclasses, json, os, sys
sys.path.insert(0, %r)
import torch
from paper_1411_1702_b200 import problems
from paper_1411_1702_b200.sampler import GpuSampler
import bench
n = int(sys.argv[1])
model = sys.argv[2]
prob = (problems.chain8(particles=n, T=8, seed=1) if model == "chain" else
        problems.robertson(particles=n, T=400, seed=1) if model == "robertson" else
        problems.lotka_volterra(particles=n, T=20, seed=1) if model == "lv" else
        problems.metabolic(particles=n, n_obs=50, seed=1))
g = GpuSampler(model, dataclasses.replace(prob.cfg, arithmetic=sys.argv[3]), prob.obs)
prob.init(g)
ms, it = bench._timed_steps(g, prob, 3, 2, torch.cuda.ExternalStream(g.stream_handle))
print(json.dumps({"ms": sum(ms) / len(ms), "newton": float(sum(it)) / len(it) / n}))
""" % ROOT


def run(lib, n, model, arith):
    env = dict(os.environ, PFSMC_GPU_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", CHILD, str(n), model, arith], env=env, capture_output=True, text=True,
                         check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


def main():
    a, b = sys.argv[1], sys.argv[2]
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    n = int(sys.argv[4]) if len(sys.argv) > 4 else 1 << 22
    model = sys.argv[5] if len(sys.argv) > 5 else "chain"
    arith = sys.argv[6] if len(sys.argv) > 6 else "exact"
    res = {a: [], b: []}
    for r in range(rounds):
        for lib in ((a, b) if r % 2 == 0 else (b, a)):
            v = run(lib, n, model, arith)
            res[lib].append(v["ms"])
            print(f"{os.path.basename(lib):>8s} {v['ms']:.3f} ms/step  newton/particle-step {v['newton']:.2f}", flush=True)
    for lib in (a, b):
        print(f"median {os.path.basename(lib):>8s} {statistics.median(res[lib]):.3f} ms/step")


if __name__ == "__main__":
    main()
