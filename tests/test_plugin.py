"""Caller-defined model plugins (include/pfsmc_gpu_model.cuh) — the open form
of the reference's OdeModel::bind -> ModelEval contract (models.hpp:20-55).

CPU: the example plugin (examples/user_model/libuser_models.so) loads and
registers its models with libpfsmc_gpu.so. GPU: a sampler created with the
plugin's id runs the plugin's kernels; the plugin's Lotka-Volterra (term for
term the built-in model) matches the C oracle's LV at the north_star bars,
and the SIR model (not shipped by the library) runs a filter."""
import os

import numpy as np
import pytest

from oracle_ctypes import Oracle, StepConfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PLUGIN = os.path.join(ROOT, "examples", "user_model", "libuser_models.so")


def _load():
    from paper_1411_1702_b200.sampler import load_model_plugin
    return load_model_plugin(PLUGIN)


def test_plugin_registers_its_models():
    got = _load()
    assert got["UserLotkaVolterra"] == (100, 2, 2)
    assert got["SirModel"] == (101, 3, 2)


@pytest.mark.gpu
@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_plugin_model_lockstep_vs_oracle(arith):
    from paper_1411_1702_b200 import problems
    from paper_1411_1702_b200.sampler import Ensemble, GpuSampler, ObservationModel, PfConfig
    _load()
    O = Oracle()
    n, steps = 1 << 14, 4
    prob = problems.lotka_volterra(particles=n, T=steps, seed=41)
    sc = StepConfig(model="lv", family="am", order=2, h=0.1, a=0.98, seed=41, obs_idx=(0, 1), sigma=0.05)
    ens = O.init_uniform("lv", n, 41, **prob.prior)
    cfg = PfConfig(particles=n, shrink_a=0.98, h=0.1, family="am", order=2, seed=41, arithmetic=arith)
    gpu = GpuSampler("UserLotkaVolterra", cfg, ObservationModel([0, 1], 0.05))
    tp = 0.0
    for j in range(1, steps + 1):
        gpu.set_ensemble(Ensemble(ens.states, ens.params_u, ens.logw, ens.mean_u, ens.cov_u))
        row = gpu.pf_step(prob.ys[j - 1], j, tp, prob.times[j - 1])
        tr, dg = O.pf_step(sc, ens, prob.ys[j - 1], j, tp, prob.times[j - 1], diag=True)
        anc = gpu.step_diagnostics()[0].astype(np.int64)
        assert np.array_equal(anc, dg["ancestors"]), j
        got = gpu.get_ensemble()
        assert np.max(np.abs(got.states - ens.states) / np.maximum(np.abs(ens.states), 1e-300)) < 1e-10, j
        t = np.concatenate([row.theta_mean, row.theta_var, row.state_mean, [row.ess]])
        np.testing.assert_allclose(t, tr, rtol=1e-8, atol=0)
        tp = prob.times[j - 1]
    gpu.close()


@pytest.mark.gpu
def test_plugin_sir_filter_runs():
    from paper_1411_1702_b200.sampler import GpuSampler, ObservationModel, PfConfig
    _load()
    n = 1 << 16
    cfg = PfConfig(particles=n, shrink_a=0.98, h=0.05, family="bdf", order=2, seed=3)
    g = GpuSampler("SirModel", cfg, ObservationModel([1], 0.01))
    g.initialize_uniform([0.2, 0.05], [0.6, 0.2], [0.98, 0.02, 0.0], [0.98, 0.02, 0.0])
    # noise-free truth beta = 0.4, gamma = 0.1 (RK4, h = 1e-3) observed at t = 1..10
    f = lambda x: np.array([-0.4 * x[0] * x[1], 0.4 * x[0] * x[1] - 0.1 * x[1], 0.1 * x[1]])
    x, ys = np.array([0.98, 0.02, 0.0]), []
    for _ in range(10):
        for _ in range(1000):
            k1 = f(x); k2 = f(x + 5e-4 * k1); k3 = f(x + 5e-4 * k2); k4 = f(x + 1e-3 * k3)
            x = x + 1e-3 / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
        ys.append(x[1])
    tp = 0.0
    for j, y in enumerate(ys, 1):
        row = g.pf_step([y], j, tp, float(j), h=0.05)
        assert np.isfinite(row.theta_mean).all() and row.ess > 1.0
        tp = float(j)
    # the posterior concentrates near the truth
    assert abs(row.theta_mean[0] - 0.4) < 0.08 and abs(row.theta_mean[1] - 0.1) < 0.04, row.theta_mean
    g.close()
