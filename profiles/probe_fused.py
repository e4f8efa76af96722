"""Timestamps of the single-pass exact scan (k_scan_fused): tile 0 start -> last tile
start / phase 1 done / look-back done / end, LV 2^20 and config 5 at 2^25."""
import ctypes as C, numpy as np, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_1702_b200 import problems
from paper_1411_1702_b200.sampler import GpuSampler, Ensemble, ObservationModel, PfConfig
ts = (C.c_uint64 * 8)()
def show(tag, h):
    h.lib.pfsmc_gpu_debug_timestamps(h.h, ts)
    t0 = ts[0]
    print(tag, "last tile start %.1f, phase1 done %.1f, look-back done %.1f, end %.1f us; tile 0 end %.1f" % (
        (ts[1] - t0) / 1e3, (ts[3] - t0) / 1e3, (ts[4] - t0) / 1e3, (ts[2] - t0) / 1e3, (ts[5] - t0) / 1e3))
prob = problems.lotka_volterra(particles=1 << 20, T=20, seed=1)
g = GpuSampler("lv", prob.cfg, prob.obs); g.initialize_uniform(**prob.prior)
tp = 0.0
for j in range(1, 9):
    g.pf_step(prob.ys[j - 1], j, tp, prob.times[j - 1]); tp = prob.times[j - 1]
    show("lv %d" % j, g)
g.close()
if "--c5" in sys.argv:
    n5 = 1 << 25
    s = GpuSampler("payload64", PfConfig(particles=n5, seed=5), ObservationModel([0], 1.0))
    rng = np.random.default_rng(0)
    s.set_ensemble(Ensemble(rng.standard_normal((n5, 6)), rng.standard_normal((n5, 2)), np.zeros(n5), np.zeros(2), np.eye(2)))
    for sigma in (1.0,):
        s.c5_set_logweights(sigma, 1)
        for it in range(3):
            s.c5_iteration(it + 1); s.synchronize()
            show("c5 sigma %g" % sigma, s)
