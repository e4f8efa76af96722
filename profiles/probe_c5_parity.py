"""Diagnose C5 ancestor mismatches vs the oracle at a ragged 4096-tile size."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from oracle_ctypes import Oracle
from paper_1411_1702_b200.sampler import Ensemble, GpuSampler, ObservationModel, PfConfig
O = Oracle()
n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 22) + 4097 * 3 + 5
rng = np.random.default_rng(3)
s = GpuSampler("payload64", PfConfig(particles=n, seed=77), ObservationModel([0], 1.0))
states = rng.standard_normal((n, 6)); params = rng.standard_normal((n, 2))
s.set_ensemble(Ensemble(states, params, np.zeros(n), np.zeros(2), np.eye(2)))
s.c5_set_logweights(1.0, 5)
lw = s.get_ensemble().logw.copy()
s.c5_iteration(1); s.synchronize()
anc, _, _ = s.step_diagnostics()
g = O.fitness(lw, np.zeros(n))
want = O.resample(g, 77, 1)
bad = np.nonzero(anc.astype(np.int64) != want)[0]
print("n", n, "mismatches", len(bad))
cdf = np.cumsum(g); cdf[-1] = max(cdf[-1], 1.0)
for b in bad[:10]:
    u = O.draws(77, 1, int(b), 3, 1, 1)[0]
    k = want[b]; k2 = anc[b]
    print(b, "u", repr(u), "oracle", k, "gpu", k2, "cdf[k-1]", repr(cdf[k - 1] if k else 0.0), "cdf[k]", repr(cdf[k]),
          "cdf[gpu]", repr(cdf[k2]), "dist", min(abs(u - cdf[max(k - 1, 0)]), abs(u - cdf[k])))
# injected-g check: the GPU exact CDF on the oracle's own g
a2, cdf2 = s.resample_from_g(g, 1, with_cdf=True)
if a2 is not None:
    print("injected-g ancestors equal:", np.array_equal(np.asarray(a2, dtype=np.int64), want),
          "cdf equal:", np.array_equal(cdf2, cdf))
s.close()
