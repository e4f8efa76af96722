"""Config 5 at 2^25, SPLIT search: the gather making the next iteration's moment sums vs the stats pass reading theta."""
import json, os, statistics, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_1702_b200.sampler import Ensemble, GpuSampler, ObservationModel, PfConfig
n = 1 << 25
s = GpuSampler("payload64", PfConfig(particles=n, seed=5), ObservationModel([0], 1.0))
rng = np.random.default_rng(0)
s.set_ensemble(Ensemble(rng.standard_normal((n, 6)), rng.standard_normal((n, 2)), np.zeros(n), np.zeros(2), np.eye(2)))
st = torch.cuda.ExternalStream(s.stream_handle)
s.c5_set_search("split")
out = {}
for sigma in (0.1, 1.0, 4.0):
    for rnd in range(2):
        for on in (True, False):
            s.c5_fuse_moments(on)
            s.c5_set_logweights(sigma, 1)
            ms = []
            for it in range(8):
                s.flush_l2()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(st):
                    a.record(st)
                s.c5_iteration(it + 1)
                with torch.cuda.stream(st):
                    b.record(st)
                s.synchronize()
                if it >= 2:
                    ms.append(a.elapsed_time(b))
            out.setdefault(f"sigma={sigma} fuse={on}", []).append(round(statistics.median(ms), 4))
print(json.dumps(out, indent=1))
