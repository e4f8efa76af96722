"""GPU parity for the reference's problem 2, AdvDiffModel (models.cpp:158-266):
the particle-per-CTA kernels (csrc/advdiff.cuh) through the C ABI against
the C oracle (itself bitwise equal to the reference, test_advdiff.py and the
golden fixtures pf_advdiff_*.npz replayed in test_gpu_parity.py).

The only non-bitwise operation is the Newton correction: the reference
factors I - h b0 L with a sparse LU, the GPU diagonalises it with the 2-D
DFT; both are exact solves, equal to rounding. Bars as everywhere:
ancestors bit-exact, states / params / weights 1e-10, trace 1e-8 — the
state bar read normwise per particle (max_k |dx_k| / max_k |x_k| over the
grid, _rel_rows), the relative error of a field whose far-field values are
near zero.
Grid sizes cover the three register widths (E = 1: d <= 128, E = 3:
d <= 384, E = 8: d <= 1024).
"""
import ctypes as C

import numpy as np
import pytest

from oracle_ctypes import METABOLIC_DEFAULTS, Oracle, StepConfig, set_advdiff_grid
from test_gpu_parity import REL_TRACE, _compare_step, _rel, _rel_rows, _sampler, _to_gpu_ens

pytestmark = pytest.mark.gpu
O = Oracle()
TRUTH = np.array([9.0, 4.0, 6.0, 2.5, -1.5])   # bench.cpp:251-255
PRIOR_MU = [np.log(7.0), np.log(5.0), 4.0, 0.0, 0.0]
PRIOR_SD = [0.35, 0.35, 2.0, 2.0, 2.0]


@pytest.fixture(autouse=True)
def _reset_consts():
    yield
    O.set_model_consts(METABOLIC_DEFAULTS)


def plume(n):
    x0 = np.zeros((n - 1) ** 2)
    O.lib.or_gaussian_plume_ic(n, x0.ctypes.data_as(C.POINTER(C.c_double)))
    return x0


def _setup(n, N, seed, sites, **kw):
    set_advdiff_grid(n, O)
    d = (n - 1) ** 2
    x0 = plume(n)
    idx = tuple(dict.fromkeys(int(v) % d for v in sites))  # distinct, in order
    sc = StepConfig(model="advdiff", a=0.98, seed=seed, obs_idx=idx, sigma=float(x0.max() / 10), **kw)
    ens = O.init_gaussian("advdiff", N, seed, PRIOR_MU, PRIOR_SD, x0, np.zeros(d), np.zeros(d, np.int32))
    return sc, ens, x0


def _obs(sc, x0, steps, h=0.01, seed=0):
    rng = np.random.default_rng(seed)
    xt, ys = x0.copy(), []
    for j in range(1, steps + 1):
        xt = O.propagate("advdiff", TRUTH, xt, j - 1.0, float(j), h, "bdf", 2)[0]
        ys.append(xt[list(sc.obs_idx)] + sc.sigma * rng.standard_normal(len(sc.obs_idx)))
    return ys


CASES = [
    # name, grid n, particles, steps, StepConfig kwargs
    ("n6_bdf2", 6, 512, 3, dict(family="bdf", order=2, h=0.05)),
    ("n6_am3", 6, 300, 3, dict(family="am", order=3, h=0.02)),
    ("n5_ab1", 5, 200, 2, dict(family="ab", order=1, h=0.002)),
    ("n12_bdf3", 12, 256, 2, dict(family="bdf", order=3, h=0.05)),      # d = 121, E = 1
    ("n20_bdf2", 20, 96, 2, dict(family="bdf", order=2, h=0.05)),       # d = 361, E = 3 (the default grid)
    ("n20_am2", 20, 64, 1, dict(family="am", order=2, h=0.1)),
    ("n6_adaptive", 6, 400, 3, dict(family="bdf", order=2, adaptive=True, rtol=1e-3)),
    ("n10_adaptive", 10, 200, 2, dict(family="bdf", order=2, adaptive=True, rtol=1e-3)),
    ("n26_bdf2", 26, 12, 1, dict(family="bdf", order=2, h=0.1)),        # d = 625, E = 8
    ("n33_bdf1_max_grid", 33, 4, 1, dict(family="bdf", order=1, h=0.25)),  # d = 1024: the largest grid
    ("n7_bdf2_one_particle", 7, 1, 2, dict(family="bdf", order=2, h=0.05)),
    ("n7_am2_ragged3", 7, 3, 2, dict(family="am", order=2, h=0.05)),
]


@pytest.mark.parametrize("name,n,N,steps,kw", CASES, ids=[c[0] for c in CASES])
def test_lockstep_advdiff(name, n, N, steps, kw):
    """Both sides start every step from the same (oracle) ensemble."""
    sc, ens, x0 = _setup(n, N, 31 + n, (3, 7, 11, 20, 24, 40, 77, 101), **kw)
    ys = _obs(sc, x0, steps)
    gpu = _sampler(sc, N, model_consts=(n,))
    for j in range(1, steps + 1):
        gpu.set_ensemble(_to_gpu_ens(ens))
        row = gpu.pf_step(ys[j - 1], j, j - 1.0, float(j), h=sc.h)
        trace_o, dg = O.pf_step(sc, ens, ys[j - 1], j, j - 1.0, float(j), diag=True)
        _compare_step(gpu, ens, trace_o, dg, row, field_state=True)
    gpu.close()


def test_free_running_advdiff():
    """No re-injection: device init, then GPU and oracle run 6 steps."""
    n, N, steps = 8, 2048, 6
    sc, ens, x0 = _setup(n, N, 77, (2, 9, 17, 30, 41), family="bdf", order=2, h=0.05)
    ys = _obs(sc, x0, steps)
    gpu = _sampler(sc, N, model_consts=(n,))
    d = (n - 1) ** 2
    gpu.initialize_gaussian(PRIOR_MU, PRIOR_SD, x0, np.zeros(d), np.zeros(d, np.int32))
    got = gpu.get_ensemble()
    # device draws: CUDA log / sincospi vs glibc (<= 2 ulp); the degenerate x0 prior is exact
    assert np.array_equal(got.states, ens.states)
    assert np.max(np.abs(got.params_u - ens.params_u)) < 1e-14 * np.max(np.abs(ens.params_u))
    assert np.max(np.abs(got.cov_u - ens.cov_u)) < 1e-12 * np.max(np.abs(ens.cov_u))
    for j in range(1, steps + 1):
        row = gpu.pf_step(ys[j - 1], j, j - 1.0, float(j))
        trace_o, dg = O.pf_step(sc, ens, ys[j - 1], j, j - 1.0, float(j), diag=True)
        anc_g, _, _ = gpu.step_diagnostics()
        assert np.array_equal(anc_g.astype(np.int64), dg["ancestors"]), f"step {j}"
        tr = np.concatenate([row.theta_mean, row.theta_var, row.state_mean, [row.ess]])
        assert _rel(tr[:10], trace_o[:10]) < REL_TRACE, j
        assert _rel_rows(tr[None, 10:-1], trace_o[None, 10:-1]) < REL_TRACE, j
        assert _rel(tr[-1:], trace_o[-1:]) < REL_TRACE, j
    got = gpu.get_ensemble()
    assert _rel_rows(got.states, ens.states) < 1e-8
    gpu.close()


def test_advdiff_32_sites_and_total_degeneracy():
    """The observation limit (32 sites) and the reference's NumericalError on
    total degeneracy (filter.cpp:149-152) at the same step as the oracle."""
    from paper_1411_1702_b200.sampler import NumericalError
    n, N = 9, 64
    sc, ens, x0 = _setup(n, N, 5, tuple(range(0, 64, 2)), family="bdf", order=2, h=0.05)
    assert len(sc.obs_idx) == 32
    ys = _obs(sc, x0, 1)
    gpu = _sampler(sc, N, model_consts=(n,))
    gpu.set_ensemble(_to_gpu_ens(ens))
    e0 = ens.copy()
    row = gpu.pf_step(ys[0], 1, 0.0, 1.0)
    trace_o, dg = O.pf_step(sc, ens, ys[0], 1, 0.0, 1.0, diag=True)
    _compare_step(gpu, ens, trace_o, dg, row, field_state=True)
    # a non-finite field in every particle: every rhs is invalid, every predictive
    # likelihood -inf, and fitness_weights throws (NUMERICAL)
    bad = e0.copy()
    bad.states[:, 3] = np.inf
    gpu.set_ensemble(_to_gpu_ens(bad))
    with pytest.raises(NumericalError):
        gpu.pf_step(ys[0], 1, 0.0, 1.0)
    from oracle_ctypes import OracleError
    with pytest.raises(OracleError) as ei:
        O.pf_step(sc, bad.copy(), ys[0], 1, 0.0, 1.0)
    assert ei.value.code == 3
    gpu.close()


def test_advdiff_config_errors():
    from paper_1411_1702_b200.sampler import ConfigError
    sc = StepConfig(model="advdiff", family="bdf", order=2, h=0.05, obs_idx=(0, 1), sigma=0.1)
    for bad in (3, 34, 7.5):
        with pytest.raises(ConfigError):
            _sampler(sc, 64, model_consts=(bad,))
    sc.obs_idx = tuple(range(33))
    with pytest.raises(ConfigError):
        _sampler(sc, 64, model_consts=(20,))
