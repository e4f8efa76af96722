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
if "--c5" in sys.argv:
    from paper_1411_1702_b200.sampler import Ensemble, ObservationModel, PfConfig
    n5 = 1 << 25
    s = GpuSampler("payload64", PfConfig(particles=n5, seed=5), ObservationModel([0], 1.0))
    rng = np.random.default_rng(0)
    s.set_ensemble(Ensemble(rng.standard_normal((n5, 6)), rng.standard_normal((n5, 2)), np.zeros(n5), np.zeros(2), np.eye(2)))
    for sigma in (0.1, 1.0, 4.0):
        s.c5_set_logweights(sigma, 1)
        for it in range(3):
            s.c5_iteration(it + 1)
            s.synchronize()
            s.lib.pfsmc_gpu_debug_timestamps(s.h, ts)
            print("c5 sigma", sigma, "scan->resolver start %.1f us, resolver %.1f us" % ((ts[1]-ts[0])/1e3, (ts[2]-ts[1])/1e3),
                  "| hdr+compose %.1f, scan %.1f, stage %.1f, walk %.1f us; windowed super-tiles %d, windows %d" % (
                  (ts[3]-ts[1])/1e3, (ts[4]-ts[3])/1e3, (ts[5]-ts[4])/1e3, (ts[6]-ts[5])/1e3, ts[7]//100000, ts[7]%100000))
