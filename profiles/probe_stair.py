import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1411_1702_b200.sampler import GpuSampler, ObservationModel, PfConfig
for nwin in (250, 257, 300):
    spread = np.zeros(1 << 16)
    spread[np.arange(nwin) * 200 + 7] = 2.0 ** (np.arange(nwin) - 1070.0)
    s = GpuSampler("lv", PfConfig(particles=len(spread), seed=99), ObservationModel([0, 1], 0.05))
    anc, cdf = s.resample_from_g(spread, 4, with_cdf=True)
    ref = np.cumsum(spread); ref[-1] = max(ref[-1], 1.0)
    bad = np.flatnonzero(cdf != ref)
    print(nwin, "bad", len(bad), bad[:5], [(cdf[i], ref[i]) for i in bad[:3]])
    s.close()
