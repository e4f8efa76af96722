"""Host-side mirror of the reference's per-step sampler API over the C ABI.

The reference (C++) exposes, in ``pfsmc::filter`` (filter.hpp:19-160):

* ``Ensemble`` (states N x d, params_u N x p, logw, mean_u, cov_u),
* ``PfConfig`` / ``IntegratorSpec`` / ``NewtonOpts`` / ``ObservationModel``,
* ``pf_step(ens, y, j, t_prev, t_obs, cfg, backend, model, obs)`` — the
  per-observation update this package replaces,
* ``run(data, cfg, backend, model, obs)`` — the observation loop.

:class:`GpuSampler` keeps the ensemble resident on one B200 and calls the
hand-written sm_100a kernels in ``libpfsmc_gpu.so`` through the C ABI
declared in ``include/pfsmc_gpu.h``. There is no CPU fallback: if the
extension is missing or no GPU is visible, construction raises.
Errors map like the reference's exception taxonomy (errors.hpp:9-25):
CONFIG -> :class:`ConfigError`, NUMERICAL -> :class:`NumericalError`.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# PFSMC_GPU_LIB: an alternative build of the same library (A/B timing of two
# builds on one box, profiles/ab.py); the default is the in-tree build.
LIB_PATH = os.environ.get("PFSMC_GPU_LIB") or os.path.join(HERE, "libpfsmc_gpu.so")

MODELS = {"decay": 0, "lv": 1, "robertson": 2, "chain": 3, "payload64": 4, "metabolic": 5, "advdiff": 6}
MODEL_DIMS = {0: (1, 1), 1: (2, 2), 2: (3, 3), 3: (8, 4), 4: (6, 2), 5: (3, 4)}
# AdvDiffModel(n) (models.cpp:185-249): grid (n-1)^2, params k1, k2 (positive), k3, c1, c2
ADVDIFF_DEFAULT_N = 20  # bench::ExperimentConfig.n (bench.hpp:20)


def model_dims(model: str, consts=None):
    """(d, p) of a compiled-in model; advdiff's d comes from its grid parameter."""
    if model == "advdiff":
        n = int(consts[0]) if consts else ADVDIFF_DEFAULT_N
        return (n - 1) * (n - 1), 5
    return MODEL_DIMS[MODELS[model]]
# models::MetabolicConstants defaults (models.hpp:67-74): lambda, c0, A0, A, t0_input, tau
METABOLIC_DEFAULTS = (1.0, 1.0, 1.0, 5.0, 2.0, 1.0)
FAMILIES = {"ab": 0, "am": 1, "bdf": 2}
LIKELIHOODS = {"gaussian": 0, "lognormal": 1}


class PfsmcError(RuntimeError):
    code = 1


class ConfigError(PfsmcError):
    code = 2


class NumericalError(PfsmcError):
    code = 3


ARITHMETIC = {"exact": 0, "fast": 1}

_ERRORS = {1: PfsmcError, 2: ConfigError, 3: NumericalError}

_dp = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)


class _Config(C.Structure):
    _fields_ = [("model", C.c_int), ("family", C.c_int), ("order", C.c_int),
                ("shrink_a", C.c_double), ("seed", C.c_uint64), ("newton_tol", C.c_double),
                ("newton_max_iter", C.c_int), ("particles", C.c_uint64),
                ("obs_indices", _u64p), ("n_obs", C.c_uint64), ("sigma", C.c_double),
                ("likelihood", C.c_int), ("device", C.c_int), ("model_consts", C.c_double * 8),
                ("adaptive", C.c_int), ("rtol", C.c_double), ("arithmetic", C.c_int)]


def model_consts_array(model: str, consts=None):
    """The C ABI's model_consts[8] (METABOLIC: MetabolicConstants order)."""
    if consts is None:
        consts = (METABOLIC_DEFAULTS if model == "metabolic" else
                  (ADVDIFF_DEFAULT_N,) if model == "advdiff" else ())
    v = list(map(float, consts)) + [0.0] * (8 - len(consts))
    return (C.c_double * 8)(*v[:8])


_lib = None


def load_library(path: str = LIB_PATH):
    """Loads the CUDA extension; raises if it is absent (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: run `python __graft_entry__.py build` "
                              "(the CUDA extension is required; there is no CPU path)")
        lib = C.CDLL(path)
        lib.pfsmc_gpu_last_error.restype = C.c_char_p
        lib.pfsmc_gpu_version.restype = C.c_char_p
        lib.pfsmc_gpu_stream.restype = C.c_void_p
        lib.pfsmc_gpu_stream.argtypes = [C.c_void_p]
        lib.pfsmc_gpu_create.argtypes = [C.POINTER(_Config), C.POINTER(C.c_void_p)]
        lib.pfsmc_gpu_destroy.argtypes = [C.c_void_p]
        for name in ("pfsmc_gpu_set_ensemble", "pfsmc_gpu_get_ensemble", "pfsmc_gpu_init_gaussian",
                     "pfsmc_gpu_init_uniform", "pfsmc_gpu_step", "pfsmc_gpu_upload_observations",
                     "pfsmc_gpu_step_resident", "pfsmc_gpu_synchronize", "pfsmc_gpu_run",
                     "pfsmc_gpu_get_step_diagnostics", "pfsmc_gpu_resample_from_g",
                     "pfsmc_gpu_set_kernel_timing", "pfsmc_gpu_kernel_times", "pfsmc_gpu_flush_l2",
                     "pfsmc_gpu_c5_set_logweights", "pfsmc_gpu_c5_iteration", "pfsmc_gpu_c5_set_search",
                     "pfsmc_gpu_c5_debug_bucket_cap", "pfsmc_gpu_set_scan_mode"):
            getattr(lib, name).restype = C.c_int
        _lib = lib
    return _lib


def load_model_plugin(path: str) -> dict:
    """Loads a caller-defined model plugin (include/pfsmc_gpu_model.cuh;
    examples/user_model/) and makes its models usable by name. Returns
    {name: (id, d, p)} of every registered plugin model."""
    lib = load_library()
    C.CDLL(path, mode=getattr(os, "RTLD_GLOBAL", 0x100))  # static initialisers register the models
    lib.pfsmc_gpu_registered_model.restype = C.c_int
    out, i = {}, 0
    while True:
        mid, d, p, name = C.c_int(), C.c_int(), C.c_int(), C.c_char_p()
        if lib.pfsmc_gpu_registered_model(i, C.byref(mid), C.byref(name), C.byref(d), C.byref(p)) != 0:
            break
        nm = name.value.decode()
        MODELS[nm] = mid.value
        MODEL_DIMS[mid.value] = (d.value, p.value)
        out[nm] = (mid.value, d.value, p.value)
        i += 1
    return out


def _ptr(a, t=_dp):
    return None if a is None else a.ctypes.data_as(t)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and a.shape != tuple(shape):
        a = a.reshape(shape)
    return a


@dataclass
class ObservationModel:
    """filter::ObservationModel (filter.hpp:30-33) + the likelihood kind."""
    indices: Sequence[int]
    sigma: float
    likelihood: str = "gaussian"


@dataclass
class PfConfig:
    """The fields of filter::PfConfig that pf_step reads (filter.hpp:50-65)."""
    particles: int = 1000
    shrink_a: float = 0.98
    h: float = 0.05
    family: str = "bdf"
    order: int = 2
    seed: int = 0
    newton_tol: float = 1e-9
    newton_max_iter: int = 20
    adaptive: bool = False  # IntegratorSpec.adaptive: variable-step BDF(1,2) (lmm.cpp:894-1019)
    rtol: float = 1e-3      # IntegratorSpec.rtol (adaptive only)
    arithmetic: str = "exact"  # "exact" (reference op order, bitwise Psi) or "fast" (FMA; within tolerance)


@dataclass
class Ensemble:
    """filter::Ensemble (filter.hpp:19-28), host AoS arrays."""
    states: np.ndarray
    params_u: np.ndarray
    logw: np.ndarray
    mean_u: np.ndarray
    cov_u: np.ndarray

    @property
    def n(self):
        return self.states.shape[0]

    def copy(self):
        return Ensemble(self.states.copy(), self.params_u.copy(), self.logw.copy(),
                        self.mean_u.copy(), self.cov_u.copy())


@dataclass
class TraceRow:
    """filter::TraceRow (filter.hpp:67-75)."""
    j: int
    t: float
    theta_mean: np.ndarray
    theta_var: np.ndarray
    state_mean: np.ndarray
    ess: float
    degeneracy_warning: bool = False


class GpuSampler:
    """One device-resident ensemble on one B200 behind the C ABI."""

    def __init__(self, model: str, cfg: PfConfig, obs: ObservationModel, device: int = 0,
                 model_consts=None):
        self.lib = load_library()
        self.model = model
        self.cfg = cfg
        self.obs = obs
        self.d, self.p = model_dims(model, model_consts)
        self._idx = np.ascontiguousarray(list(obs.indices), dtype=np.uint64)
        c = _Config(MODELS[model], FAMILIES[cfg.family], cfg.order, cfg.shrink_a, cfg.seed,
                    cfg.newton_tol, cfg.newton_max_iter, cfg.particles,
                    _ptr(self._idx, _u64p), len(self._idx), obs.sigma,
                    LIKELIHOODS[obs.likelihood], device, model_consts_array(model, model_consts),
                    int(cfg.adaptive), cfg.rtol, ARITHMETIC[cfg.arithmetic])
        h = C.c_void_p()
        self._check(self.lib.pfsmc_gpu_create(C.byref(c), C.byref(h)))
        self.h = h
        self.n = cfg.particles
        self.row_width = 2 * self.p + self.d + 1

    # -- plumbing ---------------------------------------------------------
    def _check(self, rc):
        if rc != 0:
            msg = self.lib.pfsmc_gpu_last_error().decode()
            raise _ERRORS.get(rc, PfsmcError)(msg)

    def close(self):
        if getattr(self, "h", None):
            self.lib.pfsmc_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream_handle(self) -> int:
        return self.lib.pfsmc_gpu_stream(self.h)

    # -- ensemble I/O -----------------------------------------------------
    def set_ensemble(self, ens: Ensemble):
        n, d, p = self.n, self.d, self.p
        a = [_f64(ens.states, (n, d)), _f64(ens.params_u, (n, p)), _f64(ens.logw, (n,)),
             _f64(ens.mean_u, (p,)), _f64(ens.cov_u, (p, p))]
        self._check(self.lib.pfsmc_gpu_set_ensemble(self.h, *[_ptr(x) for x in a]))

    def get_ensemble(self, out: Optional[Ensemble] = None) -> Ensemble:
        """The resident ensemble in the reference layout; `out` (C-contiguous
        float64 arrays of the right shapes) is filled in place, as the
        reference's pf_step mutates the caller's Ensemble (filter.cpp:332)."""
        n, d, p = self.n, self.d, self.p
        ok = out is not None and all(
            isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous and a.shape == sh
            for a, sh in ((out.states, (n, d)), (out.params_u, (n, p)), (out.logw, (n,)), (out.mean_u, (p,)),
                          (out.cov_u, (p, p))))
        e = out if ok else Ensemble(np.zeros((n, d)), np.zeros((n, p)), np.zeros(n), np.zeros(p), np.zeros((p, p)))
        self._check(self.lib.pfsmc_gpu_get_ensemble(self.h, _ptr(e.states), _ptr(e.params_u),
                                                     _ptr(e.logw), _ptr(e.mean_u), _ptr(e.cov_u)))
        return e

    def initialize_gaussian(self, th_mu, th_sigma, x_mean, x_std, x_clamp=None):
        cl = np.ascontiguousarray(x_clamp if x_clamp is not None else [0] * self.d, dtype=np.int32)
        a = [_f64(v) for v in (th_mu, th_sigma, x_mean, x_std)]
        self._check(self.lib.pfsmc_gpu_init_gaussian(self.h, *[_ptr(x) for x in a],
                                                      cl.ctypes.data_as(C.POINTER(C.c_int))))

    def initialize_uniform(self, th_lo, th_hi, x_lo, x_hi):
        a = [_f64(v) for v in (th_lo, th_hi, x_lo, x_hi)]
        self._check(self.lib.pfsmc_gpu_init_uniform(self.h, *[_ptr(x) for x in a]))

    # -- the drop-in ------------------------------------------------------
    def pf_step(self, y, j: int, t_prev: float, t_obs: float, h: Optional[float] = None) -> TraceRow:
        """filter::pf_step (filter.cpp:292-394) on the resident ensemble."""
        y = _f64(y)
        out = np.zeros(self.row_width)
        self._check(self.lib.pfsmc_gpu_step(self.h, _ptr(y), C.c_uint64(j), C.c_double(t_prev),
                                            C.c_double(t_obs), C.c_double(h or self.cfg.h),
                                            _ptr(out)))
        return self._row(j, t_obs, out)

    def _row(self, j, t, out, warn=False):
        p, d = self.p, self.d
        return TraceRow(j, t, out[:p].copy(), out[p:2 * p].copy(), out[2 * p:2 * p + d].copy(),
                        float(out[2 * p + d]), bool(warn))

    def upload_observations(self, ys, times, t0: float = 0.0, h: Optional[float] = None):
        ys = _f64(ys)
        times = _f64(times)
        self._T = len(times)
        self._times = times
        self._t0 = t0
        self._check(self.lib.pfsmc_gpu_upload_observations(self.h, _ptr(ys), _ptr(times),
                                                            C.c_uint64(len(times)), C.c_double(t0),
                                                            C.c_double(h or self.cfg.h)))

    def step_resident(self, j: int):
        self._check(self.lib.pfsmc_gpu_step_resident(self.h, C.c_uint64(j)))

    def synchronize(self) -> np.ndarray:
        out = np.zeros(self.row_width)
        self._check(self.lib.pfsmc_gpu_synchronize(self.h, _ptr(out)))
        return out

    def run(self, ys, times, t0: float = 0.0, h: Optional[float] = None):
        """filter::run (filter.cpp:396-443) from the current ensemble."""
        self.upload_observations(ys, times, t0, h)
        T = len(times)
        rows = np.zeros((T + 1, self.row_width))
        warn = np.zeros(T + 1, dtype=np.int32)
        self._check(self.lib.pfsmc_gpu_run(self.h, _ptr(rows), warn.ctypes.data_as(C.POINTER(C.c_int))))
        ts = [t0] + list(np.asarray(times, dtype=float))
        return [self._row(j, ts[j], rows[j], warn[j]) for j in range(T + 1)]

    # -- diagnostics / parity --------------------------------------------
    def step_diagnostics(self):
        anc = np.zeros(self.n, dtype=np.uint32)
        llb = np.zeros(self.n)
        it = C.c_uint64()
        self._check(self.lib.pfsmc_gpu_get_step_diagnostics(self.h, _ptr(anc, _u32p), _ptr(llb), C.byref(it)))
        return anc, llb, it.value

    def resample_from_g(self, g, j: int, with_cdf: bool = False):
        g = _f64(g)
        anc = np.zeros(self.n, dtype=np.uint32)
        cdf = np.zeros(self.n) if with_cdf else None
        self._check(self.lib.pfsmc_gpu_resample_from_g(self.h, _ptr(g), C.c_uint64(j), _ptr(anc, _u32p),
                                                        _ptr(cdf)))
        return (anc, cdf) if with_cdf else anc

    def set_kernel_timing(self, enable: bool):
        self._check(self.lib.pfsmc_gpu_set_kernel_timing(self.h, int(enable)))

    def kernel_times(self):
        ms = np.zeros(16)
        n = C.c_int()
        names = C.c_char_p()
        self._check(self.lib.pfsmc_gpu_kernel_times(self.h, _ptr(ms), C.byref(n), C.byref(names)))
        out = {}
        last = None
        for name, v in zip(names.value.decode().split(","), ms[:n.value].tolist()):
            if name == "-":  # an event slot without a kernel (fused scan): its gap belongs to the previous launch
                out[last] += v
            else:
                out[name] = v
                last = name
        return out

    # -- BASELINE config 5 microbenchmark (model "payload64") ------------
    def c5_set_logweights(self, sigma: float, key: int):
        self._check(self.lib.pfsmc_gpu_c5_set_logweights(self.h, C.c_double(sigma), C.c_uint64(key)))

    def c5_iteration(self, j: int):
        self._check(self.lib.pfsmc_gpu_c5_iteration(self.h, C.c_uint64(j)))

    def c5_set_search(self, mode: str, debug_bucket_cap: int = 0):
        """'guide' (slot-order search + gather) or 'bucketed' (uniforms
        partitioned by value first; include/pfsmc_gpu.h). debug_bucket_cap
        forces a small bucket capacity (spill-list test)."""
        if debug_bucket_cap:
            self._check(self.lib.pfsmc_gpu_c5_debug_bucket_cap(self.h, C.c_longlong(debug_bucket_cap)))
        self._check(self.lib.pfsmc_gpu_c5_set_search(self.h, {"guide": 0, "bucketed": 1, "split": 2}[mode]))

    def c5_fuse_moments(self, on: bool):
        """A/B and test knob: False makes every config-5 iteration's stats pass read theta itself
        (default: with the SPLIT search the gather makes the next iteration's moment sums)."""
        self.lib.pfsmc_gpu_c5_debug_fuse_moments.restype = C.c_int
        self._check(self.lib.pfsmc_gpu_c5_debug_fuse_moments(self.h, C.c_int(1 if on else 0)))

    def set_scan_mode(self, mode: str):
        """'fused' (one-kernel exact scan with decoupled look-back, the default)
        or 'two_pass' (records pass + resolver, CDF pass; include/pfsmc_gpu.h).
        Bitwise identical results."""
        self._check(self.lib.pfsmc_gpu_set_scan_mode(self.h, {"fused": 0, "two_pass": 1}[mode]))

    def transfer_bytes(self):
        """(H2D, D2H) bytes of one blocking pf_step (pfsmc_gpu_step_transfer_bytes)."""
        self.lib.pfsmc_gpu_step_transfer_bytes.restype = C.c_int
        a, b = C.c_uint64(), C.c_uint64()
        self._check(self.lib.pfsmc_gpu_step_transfer_bytes(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def flush_l2(self):
        self._check(self.lib.pfsmc_gpu_flush_l2(self.h))
