"""ctypes bindings for the two CPU checkers (TEST INFRASTRUCTURE).

* ``liboracle.so`` — the plain-C restatement ``oracle/pfsmc_oracle.c``.
* ``oracle/_ref/libpfsmc_ref.so`` — the unmodified reference sampler compiled
  from /root/reference/proj/src (oracle/Makefile), with a C-ABI harness.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's reference /
cpu_baseline legs import this module. Nothing in the product path does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libpfsmc_ref.so")

FAMILIES = {"ab": 0, "am": 1, "bdf": 2}
MODELS = {"decay": 0, "lv": 1, "robertson": 2, "chain": 3, "metabolic": 5, "advdiff": 6}
DIMS = {0: (1, 1), 1: (2, 2), 2: (3, 3), 3: (8, 4), 5: (3, 4), 6: (19 * 19, 5)}
# AdvDiffModel parameters (models.cpp:242-249): k1, k2 positive (log space); k3, c1, c2 not
ADVDIFF_POSITIVE = (True, True, False, False, False)


def set_advdiff_grid(n, *checkers):
    """Binds AdvDiffModel(n) (grid (n-1)^2) in every checker given and in DIMS."""
    DIMS[6] = ((n - 1) * (n - 1), 5)
    for c in checkers:
        c.set_model_consts((float(n),))
# models::MetabolicConstants defaults (models.hpp:67-74): lambda, c0, A0, A, t0_input, tau
METABOLIC_DEFAULTS = (1.0, 1.0, 1.0, 5.0, 2.0, 1.0)
LIKELIHOODS = {"gaussian": 0, "lognormal": 1}

_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)


def _ptr(a, t=_dp):
    if a is None:
        return None
    return a.ctypes.data_as(t)


class OrCfg(C.Structure):
    _fields_ = [("model", C.c_int), ("family", C.c_int), ("order", C.c_int),
                ("h", C.c_double), ("a", C.c_double), ("seed", C.c_uint64),
                ("newton_tol", C.c_double), ("newton_max_iter", C.c_int),
                ("obs_idx", _u64p), ("m_y", C.c_uint64), ("sigma", C.c_double),
                ("likelihood", C.c_int), ("adaptive", C.c_int), ("rtol", C.c_double)]


class RefCfg(C.Structure):
    _fields_ = [("model", C.c_int), ("family", C.c_int), ("order", C.c_int),
                ("h", C.c_double), ("a", C.c_double), ("seed", C.c_uint64),
                ("newton_tol", C.c_double), ("newton_max_iter", C.c_int),
                ("obs_idx", _u64p), ("m_y", C.c_uint64), ("sigma", C.c_double),
                ("workers", C.c_int), ("adaptive", C.c_int), ("rtol", C.c_double)]


class Ens(C.Structure):
    _fields_ = [("n", C.c_uint64), ("d", C.c_uint64), ("p", C.c_uint64),
                ("states", _dp), ("params_u", _dp), ("logw", _dp),
                ("mean_u", _dp), ("cov_u", _dp)]


class OrStepOut(C.Structure):
    _fields_ = [("trace", _dp), ("ancestors", _i64p), ("loglik_bar", _dp),
                ("g", _dp), ("gamma", _dp), ("status_new", _ip),
                ("newton_iters", _ip)]


@dataclass
class Ensemble:
    """Host mirror of filter::Ensemble (filter.hpp:19-28), AoS row-major."""
    states: np.ndarray    # (n, d)
    params_u: np.ndarray  # (n, p)
    logw: np.ndarray      # (n,)
    mean_u: np.ndarray    # (p,)
    cov_u: np.ndarray     # (p, p)

    @property
    def n(self):
        return self.states.shape[0]

    @property
    def d(self):
        return self.states.shape[1]

    @property
    def p(self):
        return self.params_u.shape[1]

    @staticmethod
    def empty(n, d, p):
        return Ensemble(np.zeros((n, d)), np.zeros((n, p)), np.zeros(n),
                        np.zeros(p), np.zeros((p, p)))

    def copy(self):
        return Ensemble(self.states.copy(), self.params_u.copy(),
                        self.logw.copy(), self.mean_u.copy(), self.cov_u.copy())

    def c_struct(self):
        for a in (self.states, self.params_u, self.logw, self.mean_u, self.cov_u):
            assert a.dtype == np.float64 and a.flags.c_contiguous
        return Ens(self.n, self.d, self.p, _ptr(self.states), _ptr(self.params_u),
                   _ptr(self.logw), _ptr(self.mean_u), _ptr(self.cov_u))


@dataclass
class StepConfig:
    """Flattened filter::PfConfig + ObservationModel (filter.hpp:30-65)."""
    model: str = "lv"
    family: str = "am"
    order: int = 2
    h: float = 0.1
    a: float = 0.98
    seed: int = 1
    newton_tol: float = 1e-9
    newton_max_iter: int = 20
    obs_idx: tuple = (0, 1)
    sigma: float = 0.05
    likelihood: str = "gaussian"
    adaptive: bool = False   # IntegratorSpec.adaptive (variable-step BDF(1,2))
    rtol: float = 1e-3       # IntegratorSpec.rtol

    @property
    def dims(self):
        return DIMS[MODELS[self.model]]


class _Base:
    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run __graft_entry__.build())")
        self.lib = C.CDLL(path)


class Oracle(_Base):
    """The C restatement."""

    def __init__(self, path=ORACLE_SO):
        super().__init__(path)
        L = self.lib
        L.or_last_error.restype = C.c_char_p
        L.or_log_likelihood.restype = C.c_double

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.or_last_error().decode())

    def _cfg(self, sc: StepConfig):
        idx = np.ascontiguousarray(sc.obs_idx, dtype=np.uint64)
        cfg = OrCfg(MODELS[sc.model], FAMILIES[sc.family], sc.order, sc.h, sc.a,
                    sc.seed, sc.newton_tol, sc.newton_max_iter, _ptr(idx, _u64p),
                    len(idx), sc.sigma, LIKELIHOODS[sc.likelihood], int(sc.adaptive), sc.rtol)
        return cfg, idx

    def philox(self, ctr, key):
        c = np.ascontiguousarray(ctr, dtype=np.uint64)
        k = np.ascontiguousarray(key, dtype=np.uint64)
        o = np.zeros(4, dtype=np.uint64)
        self.lib.or_philox4x64(_ptr(c, _u64p), _ptr(k, _u64p), _ptr(o, _u64p))
        return o

    def set_model_consts(self, k=METABOLIC_DEFAULTS):
        v = np.zeros(8)
        v[:len(k)] = k
        self.lib.or_set_model_consts(_ptr(v))

    def draws(self, seed, j, n, purpose, kind, count):
        out = np.zeros(count, dtype=np.uint64 if kind == 0 else np.float64)
        self._check(self.lib.or_stream_draws(C.c_uint64(seed), C.c_uint64(j), C.c_uint64(n),
                                             purpose, kind, C.c_uint64(count),
                                             out.ctypes.data_as(C.c_void_p)))
        return out

    def init_uniform(self, model, n, seed, th_lo, th_hi, x_lo, x_hi):
        d, p = DIMS[MODELS[model]]
        e = Ensemble.empty(n, d, p)
        arrs = [np.ascontiguousarray(v, dtype=np.float64) for v in (th_lo, th_hi, x_lo, x_hi)]
        s = e.c_struct()
        self._check(self.lib.or_init_uniform(MODELS[model], C.c_uint64(n), C.c_uint64(seed),
                                             *[_ptr(a) for a in arrs], C.byref(s)))
        return e

    def init_gaussian(self, model, n, seed, th_mu, th_sigma, x_mean, x_std, x_clamp):
        d, p = DIMS[MODELS[model]]
        e = Ensemble.empty(n, d, p)
        arrs = [np.ascontiguousarray(v, dtype=np.float64) for v in (th_mu, th_sigma, x_mean, x_std)]
        cl = np.ascontiguousarray(x_clamp, dtype=np.int32)
        s = e.c_struct()
        self._check(self.lib.or_init_gaussian(MODELS[model], C.c_uint64(n), C.c_uint64(seed),
                                              *[_ptr(a) for a in arrs], _ptr(cl, _ip), C.byref(s)))
        return e

    def pf_step(self, sc: StepConfig, ens: Ensemble, y, j, t_prev, t_obs, diag=False):
        """In-place step on ``ens``; returns (trace, diagnostics dict)."""
        cfg, _keep = self._cfg(sc)
        n, d, p = ens.n, ens.d, ens.p
        y = np.ascontiguousarray(y, dtype=np.float64)
        trace = np.zeros(2 * p + d + 1)
        dg = {}
        if diag:
            dg = dict(ancestors=np.zeros(n, np.int64), loglik_bar=np.zeros(n),
                      g=np.zeros(n), gamma=np.zeros((n, d)),
                      status_new=np.zeros(n, np.int32), newton_iters=np.zeros(n, np.int32))
        out = OrStepOut(_ptr(trace), _ptr(dg.get("ancestors"), _i64p), _ptr(dg.get("loglik_bar")),
                        _ptr(dg.get("g")), _ptr(dg.get("gamma")),
                        _ptr(dg.get("status_new"), _ip), _ptr(dg.get("newton_iters"), _ip))
        s = ens.c_struct()
        self._check(self.lib.or_pf_step(C.byref(cfg), C.byref(s), _ptr(y), C.c_uint64(j),
                                        C.c_double(t_prev), C.c_double(t_obs), C.byref(out)))
        return trace, dg

    def propagate(self, model, theta_nat, x0, t0, t1, h, family, order, tol=1e-9, max_iter=20):
        d, p = DIMS[MODELS[model]]
        st = np.zeros(d); gm = np.zeros(d)
        status = C.c_int(); iters = C.c_int()
        th = np.ascontiguousarray(theta_nat, dtype=np.float64)
        x = np.ascontiguousarray(x0, dtype=np.float64)
        self._check(self.lib.or_propagate_interval(MODELS[model], _ptr(th), _ptr(x), C.c_double(t0),
                                                   C.c_double(t1), C.c_double(h), FAMILIES[family],
                                                   order, C.c_double(tol), max_iter, _ptr(st), _ptr(gm),
                                                   C.byref(status), C.byref(iters)))
        return st, gm, status.value, iters.value

    def fitness(self, logw, loglik):
        logw = np.ascontiguousarray(logw, dtype=np.float64)
        loglik = np.ascontiguousarray(loglik, dtype=np.float64)
        g = np.zeros(len(logw))
        self._check(self.lib.or_fitness_weights(_ptr(logw), _ptr(loglik), C.c_uint64(len(g)), _ptr(g)))
        return g

    def resample(self, g, seed, j):
        g = np.ascontiguousarray(g, dtype=np.float64)
        out = np.zeros(len(g), np.int64)
        self._check(self.lib.or_resample_multinomial(_ptr(g), C.c_uint64(len(g)), C.c_uint64(seed),
                                                     C.c_uint64(j), _ptr(out, _i64p)))
        return out

    def weighted_mean_cov(self, params, w):
        params = np.ascontiguousarray(params, dtype=np.float64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        n, p = params.shape
        mean = np.zeros(p); cov = np.zeros((p, p))
        self._check(self.lib.or_weighted_mean_cov(_ptr(params), C.c_uint64(n), C.c_uint64(p), _ptr(w),
                                                  _ptr(mean), _ptr(cov)))
        return mean, cov

    def chol_psd(self, cov):
        cov = np.ascontiguousarray(cov, dtype=np.float64)
        p = cov.shape[0]
        L = np.zeros((p, p)); jit = C.c_double()
        self._check(self.lib.or_chol_psd(_ptr(cov), C.c_uint64(p), _ptr(L), C.byref(jit)))
        return L, jit.value


class Reference(_Base):
    """The unmodified reference, through oracle/ref/ref_harness.cpp."""

    def __init__(self, path=REF_SO):
        super().__init__(path)
        self.lib.ref_last_error.restype = C.c_char_p

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def _cfg(self, sc: StepConfig, workers=0):
        if sc.likelihood != "gaussian":
            raise ValueError("the reference has only the Gaussian likelihood")
        idx = np.ascontiguousarray(sc.obs_idx, dtype=np.uint64)
        cfg = RefCfg(MODELS[sc.model], FAMILIES[sc.family], sc.order, sc.h, sc.a, sc.seed,
                     sc.newton_tol, sc.newton_max_iter, _ptr(idx, _u64p), len(idx), sc.sigma, workers,
                     int(sc.adaptive), sc.rtol)
        return cfg, idx

    def philox(self, ctr, key):
        c = np.ascontiguousarray(ctr, dtype=np.uint64)
        k = np.ascontiguousarray(key, dtype=np.uint64)
        o = np.zeros(4, dtype=np.uint64)
        self._check(self.lib.ref_philox(_ptr(c, _u64p), _ptr(k, _u64p), _ptr(o, _u64p)))
        return o

    def set_model_consts(self, k=METABOLIC_DEFAULTS):
        v = np.zeros(8)
        v[:len(k)] = k
        self.lib.ref_set_model_consts(_ptr(v))

    def draws(self, seed, j, n, purpose, kind, count):
        out = np.zeros(count, dtype=np.uint64 if kind == 0 else np.float64)
        self._check(self.lib.ref_stream_draws(C.c_uint64(seed), C.c_uint64(j), C.c_uint64(n),
                                              purpose, kind, C.c_uint64(count),
                                              out.ctypes.data_as(C.c_void_p)))
        return out

    def pf_step(self, sc: StepConfig, ens: Ensemble, y, j, t_prev, t_obs, workers=0):
        cfg, _keep = self._cfg(sc, workers)
        y = np.ascontiguousarray(y, dtype=np.float64)
        trace = np.zeros(2 * ens.p + ens.d + 1)
        s = ens.c_struct()
        self._check(self.lib.ref_pf_step(C.byref(cfg), C.byref(s), _ptr(y), C.c_uint64(j),
                                         C.c_double(t_prev), C.c_double(t_obs), _ptr(trace), None))
        return trace

    def ancestors(self, sc: StepConfig, ens: Ensemble, y, j, t_prev, t_obs):
        cfg, _keep = self._cfg(sc)
        y = np.ascontiguousarray(y, dtype=np.float64)
        anc = np.zeros(ens.n, np.int64); ll = np.zeros(ens.n); g = np.zeros(ens.n)
        s = ens.c_struct()
        self._check(self.lib.ref_pf_step_ancestors(C.byref(cfg), C.byref(s), _ptr(y), C.c_uint64(j),
                                                   C.c_double(t_prev), C.c_double(t_obs),
                                                   _ptr(anc, _i64p), _ptr(ll), _ptr(g)))
        return anc, ll, g

    def init_gaussian(self, sc: StepConfig, n, th_mu, th_sigma, x_mean, x_std, x_clamp):
        cfg, _keep = self._cfg(sc)
        d, p = sc.dims
        e = Ensemble.empty(n, d, p)
        arrs = [np.ascontiguousarray(v, dtype=np.float64) for v in (th_mu, th_sigma, x_mean, x_std)]
        cl = np.ascontiguousarray(x_clamp, dtype=np.int32)
        s = e.c_struct()
        self._check(self.lib.ref_initialize_gaussian(C.byref(cfg), C.c_uint64(n), *[_ptr(a) for a in arrs],
                                                     _ptr(cl, _ip), C.byref(s)))
        return e

    def propagate(self, model, theta_nat, x0, t0, t1, h, family, order, tol=1e-9, max_iter=20):
        d, p = DIMS[MODELS[model]]
        st = np.zeros(d); gm = np.zeros(d)
        status = C.c_int(); iters = C.c_int()
        th = np.ascontiguousarray(theta_nat, dtype=np.float64)
        x = np.ascontiguousarray(x0, dtype=np.float64)
        self._check(self.lib.ref_propagate_interval(MODELS[model], _ptr(th), _ptr(x), C.c_double(t0),
                                                    C.c_double(t1), C.c_double(h), FAMILIES[family], order,
                                                    C.c_double(tol), max_iter, _ptr(st), _ptr(gm),
                                                    C.byref(status), C.byref(iters)))
        return st, gm, status.value, iters.value

    def fitness(self, logw, loglik):
        logw = np.ascontiguousarray(logw, dtype=np.float64)
        loglik = np.ascontiguousarray(loglik, dtype=np.float64)
        g = np.zeros(len(logw))
        self._check(self.lib.ref_fitness_weights(_ptr(logw), _ptr(loglik), C.c_uint64(len(g)), _ptr(g)))
        return g

    def resample(self, g, seed, j):
        g = np.ascontiguousarray(g, dtype=np.float64)
        out = np.zeros(len(g), np.int64)
        self._check(self.lib.ref_resample_multinomial(_ptr(g), C.c_uint64(len(g)), C.c_uint64(seed),
                                                      C.c_uint64(j), _ptr(out, _i64p)))
        return out

    def weighted_mean_cov(self, params, w):
        params = np.ascontiguousarray(params, dtype=np.float64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        n, p = params.shape
        mean = np.zeros(p); cov = np.zeros((p, p))
        self._check(self.lib.ref_weighted_mean_cov(_ptr(params), C.c_uint64(n), C.c_uint64(p), _ptr(w),
                                                   _ptr(mean), _ptr(cov)))
        return mean, cov

    def chol_psd(self, cov):
        cov = np.ascontiguousarray(cov, dtype=np.float64)
        p = cov.shape[0]
        L = np.zeros((p, p)); jit = C.c_double()
        self._check(self.lib.ref_chol_psd(_ptr(cov), C.c_uint64(p), _ptr(L), C.byref(jit)))
        return L, jit.value

    def time_steps(self, sc: StepConfig, ens: Ensemble, ys, t_obs, j0, t_prev0, workers):
        cfg, _keep = self._cfg(sc, workers)
        ys = np.ascontiguousarray(ys, dtype=np.float64)
        t_obs = np.ascontiguousarray(t_obs, dtype=np.float64)
        secs = C.c_double()
        s = ens.c_struct()
        self._check(self.lib.ref_time_steps(C.byref(cfg), C.byref(s), _ptr(ys), _ptr(t_obs),
                                            C.c_uint64(j0), C.c_uint64(len(t_obs)), C.c_double(t_prev0),
                                            C.byref(secs)))
        return secs.value


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
