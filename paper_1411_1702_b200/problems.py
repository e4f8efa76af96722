"""The BASELINE.json workloads: model, priors, integrator choice and seeded
synthetic observations (no dataset exists for them).

Conventions (documented in DESIGN.md):
* observation noise for row r uses the keyed stream (seed, r + 1, 0, init),
  components drawn in order — the reference generator's convention
  (bench.cpp:370-376);
* Lotka-Volterra truth is RK4 at h = 1e-3 (BASELINE config 1); the chain and
  Robertson truths use scipy's Radau at rtol 1e-10 (the reference generator
  is its own adaptive BDF at rtol 1e-8, bench.cpp:298-317);
* the reference ramps the LMM order up from 1 in every observation interval
  (lmm.cpp:478-481), so a configured order only engages with >= order
  sub-steps per interval (m = (t_obs - t_prev) / h).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .sampler import ObservationModel, PfConfig

# ---------------------------------------------------------------- host Philox
_M0, _M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
_W0, _W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
_KC = 0x7066736D632D3031
_MASK = (1 << 64) - 1


def philox4x64(ctr, key):
    """Philox4x64-10 (rng.cpp:28-41), Python integers."""
    c0, c1, c2, c3 = ctr
    k0, k1 = key
    for r in range(10):
        if r:
            k0 = (k0 + _W0) & _MASK
            k1 = (k1 + _W1) & _MASK
        p0 = _M0 * c0
        p1 = _M1 * c2
        c0, c1, c2, c3 = ((p1 >> 64) ^ c1 ^ k0) & _MASK, p1 & _MASK, ((p0 >> 64) ^ c3 ^ k1) & _MASK, p0 & _MASK
    return c0, c1, c2, c3


class HostStream:
    """RngStream (rng.cpp:43-75) on the host; used for observation noise."""

    def __init__(self, seed, j, n, purpose):
        self.key = (seed & _MASK, _KC)
        self.ctr = [0, j, n, purpose]
        self.block_index = 0
        self.lane = 4
        self.block = None
        self.spare = None

    def next_u64(self):
        if self.lane == 4:
            self.ctr[0] = self.block_index
            self.block_index += 1
            self.block = philox4x64(self.ctr, self.key)
            self.lane = 0
        w = self.block[self.lane]
        self.lane += 1
        return w

    def next_uniform(self):
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def next_normal(self):
        if self.spare is not None:
            s, self.spare = self.spare, None
            return s
        u1 = (float(self.next_u64() >> 11) + 1.0) * 2.0 ** -53
        u2 = self.next_uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        ang = 2.0 * 3.14159265358979323846 * u2
        self.spare = r * math.sin(ang)
        return r * math.cos(ang)


# ---------------------------------------------------------------- truths
def _lv_rhs(x, th):
    return np.array([th[0] * x[0] - x[0] * x[1], x[0] * x[1] - th[1] * x[1]])


def rk4_path(rhs, x0, th, times, h):
    x = np.array(x0, dtype=float)
    t = 0.0
    out = []
    for to in times:
        n = int(round((to - t) / h))
        for _ in range(n):
            k1 = rhs(x, th)
            k2 = rhs(x + 0.5 * h * k1, th)
            k3 = rhs(x + 0.5 * h * k2, th)
            k4 = rhs(x + h * k3, th)
            x = x + (h / 6.0) * (k1 + 2 * k2 + 2 * k3 + k4)
        t = to
        out.append(x.copy())
    return np.array(out)


def _robertson_rhs(t, x, k):
    return [-k[0] * x[0] + k[2] * x[1] * x[2], k[0] * x[0] - k[1] * x[1] ** 2 - k[2] * x[1] * x[2],
            k[1] * x[1] ** 2]


def _chain_rhs(t, x, th):
    f = th[0] * x[:7] / (1.0 + x[:7])
    o = np.empty(8)
    o[0] = 1.0 - f[0]
    o[1:7] = f[:6] - th[1] * x[1:7] - th[2] * x[1:7] ** 2
    o[7] = th[1] * x[6] - th[3] * x[7]
    return o


def radau_path(rhs, x0, th, times):
    from scipy.integrate import solve_ivp
    sol = solve_ivp(rhs, (0.0, float(times[-1])), x0, method="Radau", t_eval=times, args=(th,),
                    rtol=1e-10, atol=1e-14)
    return sol.y.T


# ---------------------------------------------------------------- problems
@dataclass
class Problem:
    name: str
    model: str
    cfg: PfConfig
    obs: ObservationModel
    truth: np.ndarray
    x0_truth: np.ndarray
    prior_kind: str          # "uniform" (natural box) or "gaussian" (unconstrained)
    prior: dict
    t0: float = 0.0
    substeps: int = 1        # m: LMM steps per observation interval
    times: np.ndarray = field(default=None)
    ys: np.ndarray = field(default=None)

    def h_for(self, t_prev, t_obs):
        return (t_obs - t_prev) / self.substeps

    def init(self, sampler):
        if self.prior_kind == "uniform":
            sampler.initialize_uniform(**self.prior)
        else:
            sampler.initialize_gaussian(**self.prior)


def lotka_volterra(particles=1024, T=200, seed=1, family="am", order=2) -> Problem:
    """BASELINE configs 1-2."""
    th = np.array([1.0, 0.8])
    x0 = np.array([1.2, 0.9])
    times = 0.1 * np.arange(1, T + 1)
    path = rk4_path(_lv_rhs, x0, th, times, 1e-3)
    ys = np.empty_like(path)
    for r in range(T):
        s = HostStream(seed, r + 1, 0, 0)
        ys[r] = [path[r, k] + 0.05 * s.next_normal() for k in range(2)]
    cfg = PfConfig(particles=particles, shrink_a=0.98, h=0.1, family=family, order=order, seed=seed)
    obs = ObservationModel([0, 1], 0.05)
    prior = dict(th_lo=[0.5, 0.5], th_hi=[1.5, 1.5], x_lo=[0.5, 0.5], x_hi=[1.5, 1.5])
    return Problem("lotka_volterra", "lv", cfg, obs, th, x0, "uniform", prior, 0.0, 1, times, ys)


def robertson(particles=1 << 22, T=400, seed=1, substeps=2, max_iter=4) -> Problem:
    """BASELINE config 3 (lognormal noise is an extension of the reference)."""
    k = np.array([0.04, 3e7, 1e4])
    x0 = np.array([1.0, 0.0, 0.0])
    times = np.logspace(-4, 3, T)
    path = radau_path(_robertson_rhs, x0, k, times)
    ys = np.empty((T, 2))
    for r in range(T):
        s = HostStream(seed, r + 1, 0, 0)
        ys[r] = [path[r, i] * math.exp(0.02 * s.next_normal()) for i in (0, 2)]
    cfg = PfConfig(particles=particles, shrink_a=0.99, h=times[0] / substeps, family="bdf", order=2,
                   seed=seed, newton_max_iter=max_iter)
    obs = ObservationModel([0, 2], 0.02, "lognormal")
    prior = dict(th_mu=list(np.log(k) + 0.5), th_sigma=[1.0] * 3, x_mean=list(x0), x_std=[0.0] * 3)
    return Problem("robertson", "robertson", cfg, obs, k, x0, "gaussian", prior, 0.0, substeps, times, ys)


def chain8(particles=1 << 24, T=500, seed=1, substeps=3) -> Problem:
    """BASELINE config 4 (x(0) = 0: not specified by BASELINE.json)."""
    th = np.array([2.0, 50.0, 5.0, 0.5])
    x0 = np.zeros(8)
    times = 0.1 * np.arange(1, T + 1)
    path = radau_path(_chain_rhs, x0, th, times)
    ys = np.empty((T, 3))
    for r in range(T):
        s = HostStream(seed, r + 1, 0, 0)
        ys[r] = [path[r, i] + 0.01 * s.next_normal() for i in (0, 3, 7)]
    cfg = PfConfig(particles=particles, shrink_a=0.98, h=0.1 / substeps, family="bdf", order=3, seed=seed)
    obs = ObservationModel([0, 3, 7], 0.01)
    prior = dict(th_lo=list(0.5 * th), th_hi=list(2.0 * th), x_lo=[0.0] * 8, x_hi=[0.0] * 8)
    return Problem("chain8", "chain", cfg, obs, th, x0, "uniform", prior, 0.0, substeps, times, ys)


def _metabolic_rhs(t, x, th, k=(1.0, 1.0, 1.0, 5.0, 2.0, 1.0)):
    lam, c0, A0, A, t0, tau = k
    dt = t - t0
    phi = A0 if dt <= 0.0 else A0 + A * dt * math.exp(-dt / tau)
    f1 = th[0] * x[0] / (x[0] + th[1])
    f2 = th[2] * x[1] / (x[1] + th[3])
    return [phi - f1, f1 - f2, f2 - lam * (x[2] - c0)]


def metabolic(particles=1 << 20, n_obs=50, t_end=10.0, seed=1, step=0.05, integrator=("bdf", 2)) -> Problem:
    """The reference's own problem 1 (bench.cpp:201-248 defaults): models::
    MetabolicModel with the default MetabolicConstants, truth (2, 0.5, 1, 0.8),
    x0 = (1, 1, 1), log-normal prior N(log(1.5, 0.7, 1.5, 0.5), 0.5^2), x0 ~
    N(1, 0.25^2) clamped at 0, every state observed at t_end i / n_obs with the
    generator's noise rule sigma = 0.05 max|x| (bench.cpp:346-355). The truth
    path is scipy Radau at rtol 1e-10 (the reference generator: its adaptive
    BDF at rtol 1e-8; pfsmc_gpu_generate_data reproduces that one)."""
    from scipy.integrate import solve_ivp
    th = np.array([2.0, 0.5, 1.0, 0.8])
    x0 = np.array([1.0, 1.0, 1.0])
    times = t_end * np.arange(1, n_obs + 1) / n_obs
    sol = solve_ivp(_metabolic_rhs, (0.0, float(times[-1])), x0, method="Radau", t_eval=times, args=(th,),
                    rtol=1e-10, atol=1e-14)
    path = sol.y.T
    sigma = 0.05 * float(np.max(np.abs(path)))
    ys = np.empty((n_obs, 3))
    for r in range(n_obs):
        s = HostStream(seed, r + 1, 0, 0)
        ys[r] = [path[r, i] + sigma * s.next_normal() for i in range(3)]
    substeps = int(round((times[0] - 0.0) / step))
    cfg = PfConfig(particles=particles, shrink_a=0.98, h=step, family=integrator[0], order=integrator[1], seed=seed)
    obs = ObservationModel([0, 1, 2], sigma)
    prior = dict(th_mu=list(np.log([1.5, 0.7, 1.5, 0.5])), th_sigma=[0.5] * 4, x_mean=[1.0] * 3,
                 x_std=[0.25] * 3, x_clamp=[1, 1, 1])
    return Problem("metabolic", "metabolic", cfg, obs, th, x0, "gaussian", prior, 0.0, substeps, times, ys)


# ---------------------------------------------------------------- problem 2
def gaussian_plume_ic(n):
    """models::gaussian_plume_ic (models.cpp:130-156), x varies fastest."""
    gam = [0.04, 0.08, 0.07, 0.10, 0.05, 0.06]
    xc = [0.20, 0.30, 0.40, 0.50, 0.50, 0.70]
    yc = [0.80, 0.40, 0.40, 0.50, 0.60, 0.50]
    m = n - 1
    u = np.zeros(m * m)
    for iy in range(m):
        y = iy / m
        for ix in range(m):
            x = ix / m
            u[iy * m + ix] = sum(math.exp(-((x - xc[i]) ** 2 + (y - yc[i]) ** 2) / (2.0 * gam[i] * gam[i]))
                                 / (gam[i] * 2.5066282746310002) for i in range(6))
    return u


def advdiff_operator(n, th):
    """AdvDiffModel::assemble_operator (models.cpp:251-261) as a dense matrix:
    L = -(k1^2 G11 + k1 k3 G12 + (k2^2 + k3^2) G22) + c1 B1 + c2 B2 with the
    periodic backward difference D (linalg.cpp:89-113), B1 = I (x) D, B2 = D (x) I."""
    m = n - 1
    D = np.eye(m) - np.roll(np.eye(m), -1, axis=1)
    I = np.eye(m)
    B1, B2 = np.kron(I, D), np.kron(D, I)
    k1, k2, k3, c1, c2 = th
    return (-(k1 * k1 * B1.T @ B1 + k1 * k3 * (B1.T @ B2 + B2.T @ B1) + (k2 * k2 + k3 * k3) * B2.T @ B2)
            + c1 * B1 + c2 * B2)


def advdiff(particles=5000, n=20, seed=1, step=0.05, integrator=("bdf", 2), adaptive=False, rtol=1e-3) -> Problem:
    """The reference's own problem 2 (bench.cpp:249-277 defaults): models::
    AdvDiffModel(n), truth (k1, k2, k3, c1, c2) = (9, 4, 6, 2.5, -1.5), the
    Gaussian-plume x(0) as a degenerate prior, log-normal priors on k1, k2 and
    normal priors on k3, c1, c2, observations at t = 1..30 of 20 distinct
    random sites drawn once from stream (seed, 0, 0, init), noise sigma =
    max|x0| / 50 (bench.cpp:327-355). The truth path is exact (the operator
    is linear: expm); the reference generator integrates it with its adaptive
    BDF at rtol 1e-8 (pfsmc_gpu_generate_data reproduces that one)."""
    from scipy.linalg import expm
    th = np.array([9.0, 4.0, 6.0, 2.5, -1.5])
    x0 = gaussian_plume_ic(n)
    d = x0.size
    s = HostStream(seed, 0, 0, 0)
    sites = []
    while len(sites) < 20:
        idx = int(s.next_uniform() * d)
        if idx < d and idx not in sites:
            sites.append(idx)
    times = np.arange(1, 31, dtype=float)
    E1 = expm(advdiff_operator(n, th))
    sigma = float(np.max(np.abs(x0))) / 50.0
    path, x = [], x0.copy()
    for _ in times:
        x = E1 @ x
        path.append(x.copy())
    ys = np.empty((30, 20))
    for r in range(30):
        ns = HostStream(seed, r + 1, 0, 0)
        ys[r] = [path[r][i] + sigma * ns.next_normal() for i in sites]
    cfg = PfConfig(particles=particles, shrink_a=0.98, h=step, family=integrator[0], order=integrator[1], seed=seed,
                   adaptive=adaptive, rtol=rtol)
    obs = ObservationModel(sites, sigma)
    prior = dict(th_mu=[math.log(7.0), math.log(5.0), 4.0, 0.0, 0.0], th_sigma=[0.35, 0.35, 2.0, 2.0, 2.0],
                 x_mean=list(x0), x_std=[0.0] * d, x_clamp=[0] * d)
    prob = Problem(f"advdiff_n{n}", "advdiff", cfg, obs, th, x0, "gaussian", prior, 0.0,
                   int(round(1.0 / step)), times, ys)
    prob.model_consts = (n,)
    return prob
