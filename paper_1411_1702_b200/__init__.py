"""B200-native drop-in for the reference LMM PF-SMC per-step update
(``pfsmc::filter::pf_step``, arXiv 1411.1702).

The hot path is hand-written sm_100a CUDA in ``csrc/`` behind the C ABI
``include/pfsmc_gpu.h``; this package is the host-side mirror of the
reference's sampler API (``sampler.GpuSampler``) plus the BASELINE problems.
"""
from .sampler import (ConfigError, Ensemble, GpuSampler, NumericalError, ObservationModel,  # noqa: F401
                      PfConfig, PfsmcError, TraceRow, load_library)

__all__ = ["GpuSampler", "PfConfig", "ObservationModel", "Ensemble", "TraceRow", "ConfigError",
           "NumericalError", "PfsmcError", "load_library"]
