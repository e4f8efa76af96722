import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, bench, ctypes
from paper_1411_1702_b200.sampler import Ensemble, GpuSampler, ObservationModel, PfConfig
print("before", bench.gather_peak(0))
n5 = 1 << 25
s = GpuSampler("payload64", PfConfig(particles=n5, seed=5), ObservationModel([0], 1.0))
print("with sampler alive", bench.gather_peak(0))
s.close()
print("after close", bench.gather_peak(0))
cr = ctypes.CDLL("libcudart.so.12") if False else None
