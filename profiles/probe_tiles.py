"""Per-tile timeline of k_scan_fused (library built with -DPFSMC_SCAN_TRACE)."""
import ctypes as C, numpy as np, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_1702_b200 import problems
from paper_1411_1702_b200.sampler import GpuSampler, Ensemble, ObservationModel, PfConfig

def show(tag, h, nt):
    buf = np.zeros(8 * nt, dtype=np.uint64)
    h.lib.pfsmc_gpu_debug_tile_times(h.h, buf.ctypes.data_as(C.POINTER(C.c_uint64)), C.c_int(nt))
    t = buf.reshape(nt, 8).astype(np.int64)
    t0 = t[:, 0].min()
    st, p1, lb, en = [(t[:, k] - t0) / 1e3 for k in range(4)]
    print(tag, "tiles", nt, "kernel span %.1f us" % en.max())
    print("  phase1 (start->classified): median %.1f  p90 %.1f  max %.1f" % (np.median(p1 - st), np.percentile(p1 - st, 90), (p1 - st).max()))
    print("  look-back wait:             median %.1f  p90 %.1f  max %.1f" % (np.median(lb - p1), np.percentile(lb - p1, 90), (lb - p1).max()))
    print("  values+emit:                median %.1f  p90 %.1f  max %.1f" % (np.median(en - lb), np.percentile(en - lb, 90), (en - lb).max()))
    idx = sorted(set([0, 1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 256, 257, nt - 1]))
    for i in idx:
        print("   tile %5d sm %3d start %6.1f p1 %6.1f lb %6.1f end %6.1f" % (i, t[i, 5], st[i], p1[i], lb[i], en[i]))
    sms = len(set(t[:, 5].tolist()))
    print("  distinct SMs", sms, " tiles started in first 5us:", int((st < 5).sum()))

prob = problems.lotka_volterra(particles=1 << 20, T=20, seed=1)
g = GpuSampler("lv", prob.cfg, prob.obs); g.initialize_uniform(**prob.prior)
tp = 0.0
for j in range(1, 6):
    g.pf_step(prob.ys[j - 1], j, tp, prob.times[j - 1]); tp = prob.times[j - 1]
show("lv", g, 512)
g.close()
n5 = 1 << 25
s = GpuSampler("payload64", PfConfig(particles=n5, seed=5), ObservationModel([0], 1.0))
rng = np.random.default_rng(0)
s.set_ensemble(Ensemble(rng.standard_normal((n5, 6)), rng.standard_normal((n5, 2)), np.zeros(n5), np.zeros(2), np.eye(2)))
s.c5_set_logweights(1.0, 1)
for it in range(3):
    s.c5_iteration(it + 1); s.synchronize()
show("c5", s, 8192)
