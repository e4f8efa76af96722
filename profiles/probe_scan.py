import ctypes as C, numpy as np, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_1411_1702_b200 import problems
from paper_1411_1702_b200.sampler import GpuSampler
prob=problems.lotka_volterra(particles=1<<20,T=20,seed=1)
g=GpuSampler("lv",prob.cfg,prob.obs); g.initialize_uniform(**prob.prior)
ts=(C.c_uint64*8)()
tp=0.0
for j in range(1,11):
    g.pf_step(prob.ys[j-1],j,tp,prob.times[j-1]); tp=prob.times[j-1]
    g.lib.pfsmc_gpu_debug_timestamps(g.h,ts)
    print(j, "scan->resolver start %.1f us, resolver %.1f us"%((ts[1]-ts[0])/1e3,(ts[2]-ts[1])/1e3),
          "| hdr+compose %.1f, scan %.1f, stage %.1f, walk %.1f us; windowed super-tiles %d, windows %d" % (
          (ts[3]-ts[1])/1e3, (ts[4]-ts[3])/1e3, (ts[5]-ts[4])/1e3, (ts[6]-ts[5])/1e3, ts[7]//100000, ts[7]%100000))
