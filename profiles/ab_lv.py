"""A/B of two library builds on the headline step (LV 2^20, resident CUDA-graph
step, events per step, L2 flushed between), alternating fresh processes.
    python profiles/ab_lv.py A.so B.so [rounds] [exact|fast]"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import dataclasses, json, sys, torch
sys.path.insert(0, %r)
from paper_1411_1702_b200 import problems
from paper_1411_1702_b200.sampler import GpuSampler
prob = problems.lotka_volterra(particles=1 << 20, T=60, seed=1)
g = GpuSampler("lv", dataclasses.replace(prob.cfg, arithmetic=sys.argv[1]), prob.obs)
g.initialize_uniform(**prob.prior)
g.upload_observations(prob.ys[:60], prob.times[:60], 0.0)
st = torch.cuda.ExternalStream(g.stream_handle)
for j in range(1, 6):
    g.step_resident(j)
g.synchronize()
ms = []
for j in range(6, 46):
    g.flush_l2()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        a.record(st)
    g.step_resident(j)
    with torch.cuda.stream(st):
        b.record(st)
    g.synchronize()
    ms.append(a.elapsed_time(b))
g.set_kernel_timing(True)
for j in range(46, 56):
    g.step_resident(j)
g.synchronize()
kt = g.kernel_times()
print(json.dumps({"ms": sum(ms) / len(ms), "kt": {k: v / 10 * 1000 for k, v in kt.items()}}))
''' % ROOT


def main():
    a, b = sys.argv[1], sys.argv[2]
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    arith = sys.argv[4] if len(sys.argv) > 4 else "exact"
    res = {a: [], b: []}
    for r in range(rounds):
        for lib in ((a, b) if r % 2 == 0 else (b, a)):
            env = dict(os.environ, PFSMC_GPU_LIB=os.path.abspath(lib))
            out = subprocess.run([sys.executable, "-c", CHILD, arith], env=env, capture_output=True, text=True,
                                 check=True).stdout
            d = json.loads(out.strip().splitlines()[-1])
            res[lib].append(d["ms"])
            print(f"{os.path.basename(lib):>12s} {d['ms']:.4f} ms", {k: round(v, 1) for k, v in d["kt"].items()},
                  flush=True)
    for lib in (a, b):
        print(f"median {os.path.basename(lib):>12s} {statistics.median(res[lib]):.4f} ms/step")


if __name__ == "__main__":
    main()
