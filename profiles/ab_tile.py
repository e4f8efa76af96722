import os, subprocess, sys, json, statistics
CH = r'''
import sys, json, torch
sys.path.insert(0, "%s")
import bench
from paper_1411_1702_b200 import problems
from paper_1411_1702_b200.sampler import GpuSampler
prob = problems.lotka_volterra(particles=1<<20, T=60, seed=1)
g = GpuSampler("lv", prob.cfg, prob.obs); g.initialize_uniform(**prob.prior)
g.upload_observations(prob.ys[:60], prob.times[:60], 0.0)
st = torch.cuda.ExternalStream(g.stream_handle)
for j in range(1, 6): g.step_resident(j)
g.synchronize()
ms = []
for j in range(6, 46):
    g.flush_l2()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st): a.record(st)
    g.step_resident(j)
    with torch.cuda.stream(st): b.record(st)
    g.synchronize(); ms.append(a.elapsed_time(b))
g.set_kernel_timing(True)
for j in range(46, 56): g.step_resident(j)
g.synchronize(); kt = g.kernel_times()
print(json.dumps({"ms": sum(ms)/len(ms), "kt": {k: v/10*1000 for k, v in kt.items()}}))
''' % os.getcwd()
res = {}
for r in range(3):
    for t in ("11", "12"):
        out = subprocess.run([sys.executable, "-c", CH], env=dict(os.environ, PFSMC_GPU_TILE_LOG2=t), capture_output=True, text=True).stdout
        d = json.loads(out.strip().splitlines()[-1]); res.setdefault(t, []).append(d["ms"])
        print(t, round(d["ms"], 4), {k: round(v, 1) for k, v in d["kt"].items()}, flush=True)
for t, v in res.items(): print("median", t, statistics.median(v))
