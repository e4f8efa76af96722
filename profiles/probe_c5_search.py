"""Config 5 at 2^25: one iteration per sigma with the slot-order (guide) and
the bucketed ancestor search, CUDA-event timed; for ncu launch lists.

  python profiles/probe_c5_search.py [guide|bucketed|both] [iterations]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_1702_b200.sampler import Ensemble, GpuSampler, ObservationModel, PfConfig  # noqa: E402

modes = ["guide", "bucketed", "split"] if len(sys.argv) < 2 or sys.argv[1] == "both" else [sys.argv[1]]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
n = 1 << 25
s = GpuSampler("payload64", PfConfig(particles=n, seed=5), ObservationModel([0], 1.0))
rng = np.random.default_rng(0)
s.set_ensemble(Ensemble(rng.standard_normal((n, 6)), rng.standard_normal((n, 2)), np.zeros(n), np.zeros(2), np.eye(2)))
stream = torch.cuda.ExternalStream(s.stream_handle)
for mode in modes:
    s.c5_set_search(mode)
    for sigma in (0.1, 1.0, 4.0):
        s.c5_set_logweights(sigma, 1)
        ms = []
        for it in range(iters):
            s.flush_l2()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                a.record(stream)
            s.c5_iteration(it + 1)
            with torch.cuda.stream(stream):
                b.record(stream)
            s.synchronize()
            ms.append(a.elapsed_time(b))
        print(f"{mode:9s} sigma={sigma}: " + " ".join(f"{x:.3f}" for x in ms) + " ms")
