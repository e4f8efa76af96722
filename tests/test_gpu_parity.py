"""GPU parity: the sm_100a kernels through the C ABI against the CPU oracle
(oracle/pfsmc_oracle.c, itself pinned bitwise to the reference in
test_oracle.py) and the reference-generated golden fixtures.

Bars (BASELINE.json north_star):
* ancestors: bit-exact (integer index work);
* states / params / weights: 1e-10 relative;
* posterior mean / covariance trace: 1e-8 relative.
The only device/host differences are CUDA's exp/log/sin/cos vs glibc
(<= 2 ulp), so every floating comparison below carries its tolerance.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle_ctypes import Ensemble as OEns
from oracle_ctypes import Oracle, StepConfig

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
O = Oracle()
REL_STATE = 1e-10
REL_TRACE = 1e-8


def _sampler(sc: StepConfig, n, likelihood="gaussian", model_consts=None, arithmetic="exact"):
    from paper_1411_1702_b200.sampler import GpuSampler, ObservationModel, PfConfig
    cfg = PfConfig(particles=n, shrink_a=sc.a, h=sc.h, family=sc.family, order=sc.order, seed=sc.seed,
                   newton_tol=sc.newton_tol, newton_max_iter=sc.newton_max_iter, adaptive=sc.adaptive,
                   rtol=sc.rtol, arithmetic=arithmetic)
    return GpuSampler(sc.model, cfg, ObservationModel(list(sc.obs_idx), sc.sigma, likelihood),
                      model_consts=model_consts)


def _to_gpu_ens(e):
    from paper_1411_1702_b200.sampler import Ensemble
    return Ensemble(e.states, e.params_u, e.logw, e.mean_u, e.cov_u)


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    fin = np.isfinite(a) & np.isfinite(b)
    assert np.array_equal(np.isfinite(a), np.isfinite(b))
    assert np.array_equal(a[~fin], b[~fin])
    if not fin.any():
        return 0.0
    return float(np.max(np.abs(a[fin] - b[fin]) / np.maximum(np.abs(b[fin]), 1e-300)))


def _rel_scaled(a, b):
    """Normwise relative error per column, max_i |a - b| / max_i |b| — the
    meaningful "relative" for quantities that cross zero (log-space params,
    log-weights, covariances)."""
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    if a.ndim == 1:
        a, b = a[:, None], b[:, None]
    a, b = a.reshape(a.shape[0], -1), b.reshape(b.shape[0], -1)
    return float(np.max(np.max(np.abs(a - b), axis=0) / np.maximum(np.max(np.abs(b), axis=0), 1e-300)))


# ---------------------------------------------------------------- resampling
def _g_cases(rng):
    out = {}
    for n in (1, 3, 4095, 4096, 4097, 65536, 1 << 20):
        g = np.exp(rng.standard_normal(n))
        out[f"lognormal1_{n}"] = g / g.sum()
    for s in (0.1, 4.0):
        g = np.exp(s * rng.standard_normal(1 << 16))
        out[f"lognormal{s}_65536"] = g / g.sum()
    out["uniform_1e5"] = np.full(100000, 1e-5)
    oh = np.zeros(1 << 18)
    oh[123457] = 1.0
    out["onehot_262144"] = oh
    two = np.zeros(10000)
    two[[10, 9000]] = 0.5
    out["twohot_exact"] = two
    short = np.full(5000, 0.9 / 5000)
    out["short_mass_guard"] = short
    z = np.exp(rng.standard_normal(50000))
    z[:20000] = 0.0
    z[30000:30100] = 0.0
    out["zeros_prefix"] = z / z.sum()
    tiny = np.exp(rng.standard_normal(20000))
    tiny[0] = 1e-300
    tiny[1] = 5e-324
    out["subnormal_head"] = tiny / tiny.sum()
    # every element doubles the running sum: one binade crossing (window) per
    # element, > kMaxWin in one tile -> serial tile + super-tile resolver
    stair = np.zeros(4096)
    stair[:1100] = 2.0 ** (np.arange(1100) - 1070.0)
    out["staircase_overflow"] = stair
    # > kResolveWin windows in total, <= kMaxWin per tile -> super-tile resolver
    spread = np.zeros(1 << 16)
    spread[np.arange(300) * 200 + 7] = 2.0 ** (np.arange(300) - 1070.0)
    out["staircase_spread"] = spread
    # ~120 windows spread over many tiles -> window-granular resolver
    mid = np.zeros(1 << 17)
    mid[np.arange(120) * 1000 + 3] = 2.0 ** (np.arange(120) - 110.0)
    mid[mid == 0] = 1e-40
    out["staircase_windows"] = mid
    return out


SCAN_MODES = ["fused", "two_pass"]  # pfsmc_gpu_set_scan_mode: bitwise the same CDF either way


@pytest.mark.parametrize("scan", SCAN_MODES)
def test_resample_from_injected_g_is_bit_exact(scan):
    """Kernel-level parity of resample_multinomial (filter.cpp:158-178): the
    device CDF equals the reference's sequential sum bit for bit, so the
    ancestors are identical for every fitness vector."""
    from paper_1411_1702_b200.sampler import GpuSampler, ObservationModel, PfConfig
    rng = np.random.default_rng(11)
    for name, g in _g_cases(rng).items():
        n = len(g)
        s = GpuSampler("lv", PfConfig(particles=n, seed=99), ObservationModel([0, 1], 0.05))
        s.set_scan_mode(scan)
        anc, cdf = s.resample_from_g(g, 4, with_cdf=True)
        ref_cdf = np.cumsum(g)
        ref_cdf[-1] = max(ref_cdf[-1], 1.0)
        assert np.array_equal(cdf, ref_cdf), (name, np.flatnonzero(cdf != ref_cdf)[:5])
        want = O.resample(g, 99, 4)
        assert np.array_equal(anc.astype(np.int64), want), (name, np.flatnonzero(anc != want)[:5])
        s.close()


@pytest.mark.parametrize("scan", SCAN_MODES)
def test_resample_randomized_structures_bit_exact(scan):
    """Property check over 40 seeded random fitness structures (sizes from 1
    to ~3e5, zero runs, σ up to 8 log-normal mass, subnormal and huge
    values): the device CDF is the sequential sum bit for bit and the
    ancestors are the reference's."""
    from paper_1411_1702_b200.sampler import GpuSampler, ObservationModel, PfConfig
    rng = np.random.default_rng(2024)
    for case in range(40):
        n = int(rng.choice([1, 2, 7, 255, 2048, 2049, 4096 * 3 + 1, int(rng.integers(1, 300000))]))
        g = np.exp(rng.uniform(0, 8) * rng.standard_normal(n) - rng.uniform(0, 700))
        if rng.random() < 0.5:
            z0 = int(rng.integers(0, n))
            g[z0:z0 + int(rng.integers(0, n))] = 0.0
        if rng.random() < 0.3:
            g[rng.integers(0, n, size=max(1, n // 50))] = 5e-324 * rng.integers(1, 1000)
        if rng.random() < 0.2:
            g[int(rng.integers(0, n))] = 2.0 ** int(rng.integers(-60, 60))
        if rng.random() < 0.5 and g.sum() > 0:
            g = g / g.sum()
        s = GpuSampler("lv", PfConfig(particles=n, seed=7 + case), ObservationModel([0, 1], 0.05))
        s.set_scan_mode(scan)
        anc, cdf = s.resample_from_g(g, 3, with_cdf=True)
        ref = np.cumsum(g)
        ref[-1] = max(ref[-1], 1.0)
        assert np.array_equal(cdf, ref), (case, n, np.flatnonzero(cdf != ref)[:5])
        want = O.resample(g, 7 + case, 3)
        assert np.array_equal(anc.astype(np.int64), want), (case, n)
        s.close()


@pytest.mark.parametrize("scan", SCAN_MODES)
def test_resample_at_config5_full_size_bit_exact(scan):
    """BASELINE config 5's per-GPU size (2^25): the device CDF is the sequential
    sum bit for bit (8192 tiles of 4096: long look-back chains / the resolver's
    super-tile path) and the ancestors are the reference's, for sigma = 4
    log-normal mass and for a vector with a long zero run and a heavy element."""
    from paper_1411_1702_b200.sampler import GpuSampler, ObservationModel, PfConfig
    n = 1 << 25
    rng = np.random.default_rng(25)
    s = GpuSampler("payload64", PfConfig(particles=n, seed=31), ObservationModel([0], 1.0))
    s.set_scan_mode(scan)
    g1 = np.exp(4.0 * rng.standard_normal(n))
    g1 /= g1.sum()
    g2 = np.exp(rng.standard_normal(n) - 30.0)
    g2[n // 3: n // 3 + (1 << 21)] = 0.0
    g2[n // 2] = 0.75
    for name, g in (("sigma4", g1), ("zeros+heavy", g2)):
        anc, cdf = s.resample_from_g(g, 2, with_cdf=True)
        ref = np.cumsum(g)
        ref[-1] = max(ref[-1], 1.0)
        assert np.array_equal(cdf, ref), (name, np.flatnonzero(cdf != ref)[:5])
        want = O.resample(g, 31, 2)
        assert np.array_equal(anc.astype(np.int64), want), name
    s.close()


@pytest.mark.parametrize("scan", SCAN_MODES)
def test_resample_golden_fixture(scan):
    from paper_1411_1702_b200.sampler import GpuSampler, ObservationModel, PfConfig
    d = np.load(os.path.join(GOLD, "resample.npz"))
    for k in [x[:-2] for x in d.files if x.endswith("_g")]:
        g = d[f"{k}_g"]
        s = GpuSampler("lv", PfConfig(particles=len(g), seed=99), ObservationModel([0, 1], 0.05))
        s.set_scan_mode(scan)
        assert np.array_equal(s.resample_from_g(g, 4).astype(np.int64), d[f"{k}_anc"]), k
        s.close()


def test_cumsum_is_sequential():
    # the check above relies on np.cumsum being the left-to-right sum
    g = np.random.default_rng(0).random(1000)
    acc, out = 0.0, []
    for v in g:
        acc += v
        out.append(acc)
    assert np.array_equal(np.cumsum(g), np.array(out))


def _rel_rows(a, b):
    """Normwise relative error per particle, max_k |a - b| / max_k |b| over a
    state vector: the relative error of a field state (the advection-diffusion
    model's d = (n-1)^2 grid values, many of them near zero)."""
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return float(np.max(np.max(np.abs(a - b), axis=1) / np.maximum(np.max(np.abs(b), axis=1), 1e-300)))


# ---------------------------------------------------------------- lock-step
def _compare_step(gpu, ens_o, trace_o, dg, row, field_state=False):
    anc_g, llb_g, _ = gpu.step_diagnostics()
    got = gpu.get_ensemble()
    mism = np.flatnonzero(anc_g.astype(np.int64) != dg["ancestors"])
    assert mism.size == 0, f"ancestor mismatch at slots {mism[:10]}"
    assert _rel(llb_g, dg["loglik_bar"]) < REL_STATE
    assert (_rel_rows if field_state else _rel)(got.states, ens_o.states) < REL_STATE
    assert _rel_scaled(got.params_u, ens_o.params_u) < REL_STATE
    w_g, w_o = np.exp(got.logw), np.exp(ens_o.logw)
    assert _rel_scaled(w_g, w_o) < REL_STATE
    assert _rel(got.mean_u, ens_o.mean_u) < REL_TRACE
    # a posterior collapsed onto one particle has a covariance of pure rounding
    # noise (the reference's two-pass sum: ~1e-26 .. 1e-90; the device's shifted
    # moments: exact 0); below 1e-20 of the parameter scale squared it is compared
    # as such, otherwise normwise at the trace bar
    floor = 1e-20 * max(1.0, float(np.max(np.abs(ens_o.params_u)))) ** 2
    if np.max(np.abs(ens_o.cov_u)) < floor:
        assert np.max(np.abs(got.cov_u)) < floor
    else:
        assert _rel_scaled(got.cov_u, ens_o.cov_u) < REL_TRACE
    tr = np.concatenate([row.theta_mean, row.theta_var, row.state_mean, [row.ess]])
    if field_state:  # the state mean of a field normwise (its entries cross zero), the rest per entry
        p, d = len(row.theta_mean), len(row.state_mean)
        assert _rel(tr[:p], trace_o[:p]) < REL_TRACE
        if np.max(np.abs(trace_o[p:2 * p])) < floor:  # collapsed posterior (see cov_u above)
            assert np.max(np.abs(tr[p:2 * p])) < floor
        else:
            assert _rel(tr[p:2 * p], trace_o[p:2 * p]) < REL_TRACE
        assert _rel_rows(tr[None, 2 * p:2 * p + d], trace_o[None, 2 * p:2 * p + d]) < REL_TRACE
        assert _rel(tr[-1:], trace_o[-1:]) < REL_TRACE
    else:
        assert _rel(tr, trace_o) < REL_TRACE


LOCKSTEP = [
    ("lv_am2_m1", dict(model="lv", family="am", order=2, h=0.1, seed=21), 1 << 16, 8, 1),
    ("lv_ab2_m1", dict(model="lv", family="ab", order=2, h=0.1, seed=22), 1 << 14, 6, 1),
    ("lv_bdf3_m4", dict(model="lv", family="bdf", order=3, h=0.025, seed=23), 1 << 13, 5, 4),
    ("lv_am3_m4", dict(model="lv", family="am", order=3, h=0.025, seed=24), 1 << 13, 5, 4),
    ("lv_ab3_m4", dict(model="lv", family="ab", order=3, h=0.025, seed=25), 1 << 13, 5, 4),
    # ragged sizes: partial warps / blocks / tiles / segments
    ("lv_am2_n5003", dict(model="lv", family="am", order=2, h=0.1, seed=26), 5003, 5, 1),
    ("lv_bdf2_n257", dict(model="lv", family="bdf", order=2, h=0.05, seed=27), 257, 5, 2),
    ("lv_am1_n3", dict(model="lv", family="am", order=1, h=0.1, seed=28), 3, 4, 1),
    ("lv_bdf1_n1", dict(model="lv", family="bdf", order=1, h=0.1, seed=30), 1, 3, 1),
    ("lv_ab2_n70001", dict(model="lv", family="ab", order=2, h=0.1, seed=29), 70001, 3, 1),
]


LOCKSTEP_FAST = [("fast_" + c[0], *c[1:]) for c in LOCKSTEP if c[0] in ("lv_am2_m1", "lv_bdf3_m4", "lv_am2_n5003")]


@pytest.mark.parametrize("name,kw,n,steps,m", LOCKSTEP + LOCKSTEP_FAST, ids=[c[0] for c in LOCKSTEP + LOCKSTEP_FAST])
def test_lockstep_lotka_volterra(name, kw, n, steps, m):
    """Both sides start every step from the same (oracle) ensemble. The
    fast_* cases run the FMA variant (PFSMC_GPU_ARITH_FAST) at the same bars."""
    from paper_1411_1702_b200 import problems
    sc = StepConfig(**kw, obs_idx=(0, 1), sigma=0.05)
    prob = problems.lotka_volterra(particles=n, T=steps, seed=kw["seed"])
    ens = O.init_uniform("lv", n, kw["seed"], **prob.prior)
    gpu = _sampler(sc, n, arithmetic="fast" if name.startswith("fast_") else "exact")
    tp = 0.0
    for j in range(1, steps + 1):
        gpu.set_ensemble(_to_gpu_ens(ens))
        t1 = prob.times[j - 1]
        row = gpu.pf_step(prob.ys[j - 1], j, tp, t1, h=(t1 - tp) / m)
        sc.h = (t1 - tp) / m
        trace_o, dg = O.pf_step(sc, ens, prob.ys[j - 1], j, tp, t1, diag=True)
        _compare_step(gpu, ens, trace_o, dg, row)
        tp = t1
    gpu.close()


def _golden_cases():
    return sorted(f[3:-4] for f in os.listdir(GOLD) if f.startswith("pf_") and f.endswith(".npz"))


@pytest.mark.parametrize("case", _golden_cases())
def test_against_reference_fixtures(case):
    """Lock-step against fixtures written by the unmodified reference."""
    d = np.load(os.path.join(GOLD, f"pf_{case}.npz"))
    kw = json.loads(str(d["config"]))
    sc = StepConfig(**kw)
    n = int(d["n"])
    gpu = _sampler(sc, n, model_consts=tuple(d["model_consts"]) if "model_consts" in d.files else None)
    ens = OEns(d["init_states"], d["init_params_u"], d["init_logw"], d["init_mean_u"], d["init_cov_u"])
    for j, (t0, t1, h) in enumerate(d["steps"], 1):
        gpu.set_ensemble(_to_gpu_ens(ens))
        row = gpu.pf_step(d["ys"][j - 1], j, float(t0), float(t1), h=float(h))
        nxt = OEns(d[f"s{j}_states"], d[f"s{j}_params_u"], d[f"s{j}_logw"], d[f"s{j}_mean_u"], d[f"s{j}_cov_u"])
        dg = {"ancestors": d[f"s{j}_anc"], "loglik_bar": d[f"s{j}_llbar"]}
        _compare_step(gpu, nxt, d[f"s{j}_trace"], dg, row, field_state=sc.model == "advdiff")
        ens = nxt
    gpu.close()


def test_free_running_lotka_volterra():
    """No re-injection: GPU and oracle run 30 steps independently."""
    from paper_1411_1702_b200 import problems
    n, steps = 1 << 14, 30
    prob = problems.lotka_volterra(particles=n, T=steps, seed=5)
    sc = StepConfig(model="lv", family="am", order=2, h=0.1, seed=5, obs_idx=(0, 1), sigma=0.05)
    ens = O.init_uniform("lv", n, 5, **prob.prior)
    gpu = _sampler(sc, n)
    gpu.set_ensemble(_to_gpu_ens(ens))
    tp = 0.0
    for j in range(1, steps + 1):
        t1 = prob.times[j - 1]
        row = gpu.pf_step(prob.ys[j - 1], j, tp, t1)
        trace_o, dg = O.pf_step(sc, ens, prob.ys[j - 1], j, tp, t1, diag=True)
        anc_g, _, _ = gpu.step_diagnostics()
        assert np.array_equal(anc_g.astype(np.int64), dg["ancestors"]), f"step {j}"
        tr = np.concatenate([row.theta_mean, row.theta_var, row.state_mean, [row.ess]])
        assert _rel(tr, trace_o) < REL_TRACE, j
        tp = t1
    got = gpu.get_ensemble()
    assert _rel(got.states, ens.states) < 1e-8
    gpu.close()


# ---------------------------------------------------------------- stiff models
@pytest.mark.parametrize("th0", [2.0, 120.0])
def test_lockstep_chain_bdf3(th0):
    # th0 = 120: h b0 dflux beats the diagonal, so the Newton LU pivots and
    # the banded solve must hand over to the dense one (lmm.cuh band_solve)
    th = np.array([th0, 50.0, 5.0, 0.5])
    n = 4096
    sc = StepConfig(model="chain", family="bdf", order=3, h=0.1 / 3, a=0.98, seed=8, obs_idx=(0, 3, 7), sigma=0.01)
    ens = O.init_uniform("chain", n, 8, 0.5 * th, 2 * th, [0] * 8, [0] * 8)
    gpu = _sampler(sc, n)
    rng = np.random.default_rng(3)
    tp = 0.0
    for j in range(1, 5):
        y = np.array([0.09 * j, 0.001 * j, 0.0]) + 0.01 * rng.standard_normal(3)
        gpu.set_ensemble(_to_gpu_ens(ens))
        row = gpu.pf_step(y, j, tp, tp + 0.1)
        trace_o, dg = O.pf_step(sc, ens, y, j, tp, tp + 0.1, diag=True)
        _compare_step(gpu, ens, trace_o, dg, row)
        tp += 0.1
    gpu.close()


@pytest.mark.parametrize("family,order,consts", [("bdf", 2, None), ("am", 3, None),
                                                 ("bdf", 3, (0.7, 0.5, 1.2, 3.0, 1.9, 0.6))])
def test_lockstep_metabolic(family, order, consts):
    """The reference's own problem-1 model (models.cpp:37-119): time-dependent
    input flux, constants bound at creation, Gaussian prior with clamped x0;
    intervals straddle the input switch-on at t0_input, m = 4 sub-steps."""
    n = 6000
    k = consts or (1.0, 1.0, 1.0, 5.0, 2.0, 1.0)
    O.set_model_consts(k)
    try:
        sc = StepConfig(model="metabolic", family=family, order=order, h=0.05, a=0.98, seed=12,
                        obs_idx=(0, 1, 2), sigma=0.1)
        mu = np.log([1.5, 0.7, 1.5, 0.5])
        ens = O.init_gaussian("metabolic", n, 12, mu, [0.5] * 4, [1.0] * 3, [0.25] * 3, [1, 1, 1])
        gpu = _sampler(sc, n, model_consts=k)
        rng = np.random.default_rng(8)
        tp = 1.6
        for j in range(1, 6):
            y = np.array([1.0, 1.2, 1.1]) + 0.1 * rng.standard_normal(3)
            gpu.set_ensemble(_to_gpu_ens(ens))
            row = gpu.pf_step(y, j, tp, tp + 0.2)
            trace_o, dg = O.pf_step(sc, ens, y, j, tp, tp + 0.2, diag=True)
            _compare_step(gpu, ens, trace_o, dg, row)
            tp += 0.2
        gpu.close()
    finally:
        O.set_model_consts((1.0, 1.0, 1.0, 5.0, 2.0, 1.0))


@pytest.mark.parametrize("model,rtol", [("metabolic", 1e-3), ("metabolic", 1e-5), ("lv", 1e-4),
                                        ("robertson", 1e-3)])
def test_lockstep_adaptive_bdf(model, rtol):
    """Variable-step BDF(1,2) (adaptive_bdf_interval, lmm.cpp:894-1019): per-
    particle step-size control, Newton corrector, gamma = rtol * steps."""
    rng = np.random.default_rng(9)
    n = 5000
    if model == "metabolic":
        sc = StepConfig(model=model, family="bdf", order=2, seed=6, obs_idx=(0, 1, 2), sigma=0.1,
                        adaptive=True, rtol=rtol)
        mu = np.log([1.5, 0.7, 1.5, 0.5])
        ens = O.init_gaussian(model, n, 6, mu, [0.5] * 4, [1.0] * 3, [0.25] * 3, [1, 1, 1])
        ys = [np.array([1.0, 1.2, 1.1]) + 0.1 * rng.standard_normal(3) for _ in range(4)]
        ts = [1.6 + 0.2 * k for k in range(5)]
    elif model == "lv":
        sc = StepConfig(model=model, family="bdf", order=2, seed=6, adaptive=True, rtol=rtol)
        ens = O.init_uniform("lv", n, 6, [0.5, 0.5], [1.5, 1.5], [0.5, 0.5], [1.5, 1.5])
        ys = [np.array([1.2, 0.9]) + 0.05 * rng.standard_normal(2) for _ in range(4)]
        ts = [0.1 * k for k in range(5)]
    else:
        sc = StepConfig(model=model, family="bdf", order=2, a=0.99, seed=6, obs_idx=(0, 2), sigma=0.02,
                        newton_max_iter=4, adaptive=True, rtol=rtol)
        ens = O.init_gaussian(model, n, 6, np.log([0.04, 3e7, 1e4]) + 0.5, [1, 1, 1], [1, 0, 0], [0, 0, 0],
                              [0, 0, 0])
        ts = [0.0] + list(np.logspace(-4, 3, 400)[:4])
        ys = [np.array([1 - 0.04 * t, 0.04 * t * 1e-3]) + 1e-3 * rng.standard_normal(2) for t in ts[1:]]
    gpu = _sampler(sc, n)
    for j in range(1, len(ts)):
        gpu.set_ensemble(_to_gpu_ens(ens))
        row = gpu.pf_step(ys[j - 1], j, ts[j - 1], ts[j])
        trace_o, dg = O.pf_step(sc, ens, ys[j - 1], j, ts[j - 1], ts[j], diag=True)
        _compare_step(gpu, ens, trace_o, dg, row)
    gpu.close()


def test_metabolic_config_error():
    """tau <= 0 is a ConfigError at model construction (models.cpp:104-108)."""
    from paper_1411_1702_b200.sampler import NumericalError
    sc = StepConfig(model="metabolic", family="bdf", order=2, h=0.05, obs_idx=(0, 1, 2), sigma=0.1)
    with pytest.raises(Exception) as e:
        _sampler(sc, 64, model_consts=(1.0, 1.0, 1.0, 5.0, 2.0, 0.0))
    assert "tau" in str(e.value) and not isinstance(e.value, NumericalError)


def test_lockstep_robertson_lognormal():
    from paper_1411_1702_b200 import problems
    n = 4096
    prob = problems.robertson(particles=n, T=400, seed=4)  # first 6 of the 400 log-spaced times
    sc = StepConfig(model="robertson", family="bdf", order=2, a=0.99, seed=4, obs_idx=(0, 2), sigma=0.02,
                    newton_max_iter=4, likelihood="lognormal")
    ens = O.init_gaussian("robertson", n, 4, prob.prior["th_mu"], prob.prior["th_sigma"], prob.prior["x_mean"],
                          prob.prior["x_std"], [0, 0, 0])
    gpu = _sampler(sc, n, likelihood="lognormal")
    tp = 0.0
    for j in range(1, 7):
        t1 = prob.times[j - 1]
        sc.h = (t1 - tp) / 2
        gpu.set_ensemble(_to_gpu_ens(ens))
        row = gpu.pf_step(prob.ys[j - 1], j, tp, t1, h=sc.h)
        trace_o, dg = O.pf_step(sc, ens, prob.ys[j - 1], j, tp, t1, diag=True)
        _compare_step(gpu, ens, trace_o, dg, row)
        tp = t1
    gpu.close()


# ---------------------------------------------------------------- init / errors
def test_device_initialisation_matches_oracle():
    from paper_1411_1702_b200 import problems
    n = 10000
    prob = problems.lotka_volterra(particles=n, T=1, seed=9)
    gpu = _sampler(StepConfig(model="lv", seed=9), n)
    gpu.initialize_uniform(**prob.prior)
    got = gpu.get_ensemble()
    ens = O.init_uniform("lv", n, 9, **prob.prior)
    assert np.array_equal(got.states, ens.states)        # uniforms are integer-exact
    assert _rel_scaled(got.params_u, ens.params_u) < 1e-14  # log: CUDA vs glibc
    assert np.array_equal(got.logw, ens.logw)
    assert _rel(got.mean_u, ens.mean_u) < 1e-12
    assert _rel_scaled(got.cov_u, ens.cov_u) < 1e-10
    gpu.close()
    sc = StepConfig(model="robertson", seed=9, obs_idx=(0, 2), sigma=0.02)
    gpu = _sampler(sc, n)
    mu = list(np.log([0.04, 3e7, 1e4]) + 0.5)
    gpu.initialize_gaussian(mu, [1, 1, 1], [1, 0, 0], [0, 0, 0])
    got = gpu.get_ensemble()
    ens = O.init_gaussian("robertson", n, 9, mu, [1, 1, 1], [1, 0, 0], [0, 0, 0], [0, 0, 0])
    assert _rel_scaled(got.params_u, ens.params_u) < 1e-13  # normals: CUDA log/sin/cos
    assert np.array_equal(got.states, ens.states)
    gpu.close()


def test_total_degeneracy_raises_numerical_at_same_step():
    from paper_1411_1702_b200.sampler import NumericalError
    n = 2048
    sc = StepConfig(model="lv", family="am", order=2, h=0.1, seed=2, obs_idx=(0, 1), sigma=0.05)
    ens = O.init_uniform("lv", n, 2, [0.5, 0.5], [1.5, 1.5], [0.5, 0.5], [1.5, 1.5])
    gpu = _sampler(sc, n)
    gpu.set_ensemble(_to_gpu_ens(ens))
    with pytest.raises(NumericalError, match="total degeneracy"):
        gpu.pf_step(np.array([1e200, 1e200]), 1, 0.0, 0.1)
    gpu.close()


def test_queued_step_error_is_sticky():
    """A failure inside a run of non-blocking resident steps (step 3 of 5: an
    observation no particle can explain) surfaces at the next synchronize and
    is not wiped by the steps queued after it; the ensemble stays at step 2's
    (later steps early-exit), like filter::run throwing at that step."""
    from paper_1411_1702_b200.sampler import NumericalError
    n = 4096
    sc = StepConfig(model="lv", family="am", order=2, h=0.1, seed=2, obs_idx=(0, 1), sigma=0.05)
    ens = O.init_uniform("lv", n, 2, [0.5, 0.5], [1.5, 1.5], [0.5, 0.5], [1.5, 1.5])
    ys = np.array([[1.1, 0.9], [1.0, 0.95], [1e200, 1e200], [1.0, 1.0], [1.0, 1.0]])
    ts = 0.1 * np.arange(1, 6)
    gpu = _sampler(sc, n)
    gpu.set_ensemble(_to_gpu_ens(ens))
    gpu.upload_observations(ys, ts, 0.0)
    gpu.step_resident(1)
    gpu.step_resident(2)
    gpu.synchronize()
    after2 = gpu.get_ensemble()
    for j in (3, 4, 5):
        gpu.step_resident(j)
    with pytest.raises(NumericalError, match="total degeneracy"):
        gpu.synchronize()
    got = gpu.get_ensemble()
    assert np.array_equal(got.states, after2.states) and np.array_equal(got.params_u, after2.params_u)
    gpu.synchronize()  # reported once: the word is clear again
    gpu.pf_step(ys[3], 4, 0.2, 0.3)  # and the filter continues from step 2
    gpu.close()


def test_shard_handle_rejects_single_handle_step():
    from paper_1411_1702_b200.sampler import ConfigError, PfConfig, ObservationModel
    from paper_1411_1702_b200.sharded import GpuShard
    sh = GpuShard("lv", PfConfig(particles=1 << 15, seed=1), ObservationModel([0, 1], 0.05), 0, 2)
    with pytest.raises(ConfigError):
        sh.pf_step([1.0, 1.0], 1, 0.0, 0.1)
    # the C ABI refuses it too (not just the Python override)
    import ctypes as C
    y = np.array([1.0, 1.0])
    out = np.zeros(8)
    rc = sh.lib.pfsmc_gpu_step(sh.h, y.ctypes.data_as(C.POINTER(C.c_double)), C.c_uint64(1), C.c_double(0.0),
                               C.c_double(0.1), C.c_double(0.1), out.ctypes.data_as(C.POINTER(C.c_double)))
    assert rc == 2
    sh.close()


def test_config_errors():
    from paper_1411_1702_b200.sampler import ConfigError
    with pytest.raises(ConfigError):
        _sampler(StepConfig(model="lv", a=1.0), 16)
    with pytest.raises(ConfigError):
        _sampler(StepConfig(model="lv", obs_idx=(0, 0)), 16)
    gpu = _sampler(StepConfig(model="lv"), 16)
    gpu.initialize_uniform([0.5, 0.5], [1.5, 1.5], [0.5, 0.5], [1.5, 1.5])
    with pytest.raises(ConfigError, match="integer step count"):
        gpu.pf_step([1.0, 1.0], 1, 0.0, 0.1, h=0.03)
    # the scan-mode knob: unknown modes are CONFIG; the kernel-time slots are named per mode
    assert gpu.lib.pfsmc_gpu_set_scan_mode(gpu.h, 7) == ConfigError.code
    assert "k_scan_fused" in gpu.kernel_times() and "k_scan_cdf" not in gpu.kernel_times()
    gpu.set_scan_mode("two_pass")
    assert {"k_scan_pieces", "k_scan_cdf"} <= set(gpu.kernel_times())
    gpu.close()


def test_run_matches_oracle_loop():
    """filter::run semantics: row 0 + T rows, degeneracy streak flags."""
    from paper_1411_1702_b200 import problems
    n, T = 1024, 20
    prob = problems.lotka_volterra(particles=n, T=T, seed=1)
    sc = StepConfig(model="lv", family="am", order=2, h=0.1, seed=1, obs_idx=(0, 1), sigma=0.05)
    ens = O.init_uniform("lv", n, 1, **prob.prior)
    gpu = _sampler(sc, n)
    gpu.set_ensemble(_to_gpu_ens(ens))
    rows = gpu.run(prob.ys, prob.times)
    assert len(rows) == T + 1 and rows[0].j == 0 and rows[-1].j == T
    tp = 0.0
    for j in range(1, T + 1):
        trace_o, _ = O.pf_step(sc, ens, prob.ys[j - 1], j, tp, prob.times[j - 1])
        r = rows[j]
        tr = np.concatenate([r.theta_mean, r.theta_var, r.state_mean, [r.ess]])
        assert _rel(tr, trace_o) < REL_TRACE, j
        tp = prob.times[j - 1]
    gpu.close()


def test_baseline_config1_full_run_vs_reference():
    """BASELINE config 1 end to end: LV, N = 1024, all T = 200 observations,
    the GPU's filter::run (one graph per step) against the unmodified
    reference's pf_step loop (oracle/_ref), free running from the same
    ensemble: every posterior mean / variance / ESS row within 1e-8."""
    from oracle_ctypes import REF_SO, Reference
    from paper_1411_1702_b200 import problems
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    R = Reference()
    n, T = 1024, 200
    prob = problems.lotka_volterra(particles=n, T=T, seed=1)
    sc = StepConfig(model="lv", family="am", order=2, h=0.1, seed=1, obs_idx=(0, 1), sigma=0.05)
    ens = O.init_uniform("lv", n, 1, **prob.prior)
    gpu = _sampler(sc, n)
    gpu.set_ensemble(_to_gpu_ens(ens))
    rows = gpu.run(prob.ys, prob.times)
    tp, worst = 0.0, 0.0
    for j in range(1, T + 1):
        trace_r = R.pf_step(sc, ens, prob.ys[j - 1], j, tp, prob.times[j - 1])
        r = rows[j]
        tr = np.concatenate([r.theta_mean, r.theta_var, r.state_mean, [r.ess]])
        worst = max(worst, _rel(tr, trace_r))
        assert worst < REL_TRACE, (j, worst)
        tp = prob.times[j - 1]
    gpu.close()


def test_cpp_drop_in_example_matches_oracle():
    """The C++ mirror (include/pfsmc_gpu.hpp) used as a pf_step call-site
    replacement: trace rows agree with the oracle run from the same prior."""
    import subprocess
    from paper_1411_1702_b200 import problems
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "examples", "drop_in_lv")
    n, T, seed = 4096, 5, 7
    prob = problems.lotka_volterra(particles=n, T=T, seed=seed)
    inp = "\n".join(f"{float(a)!r} {float(b)!r}" for a, b in prob.ys) + "\n"
    out = subprocess.run([exe, str(n), str(T), str(seed)], input=inp, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    rows = [list(map(float, ln.split()[1:])) for ln in out.stdout.strip().splitlines()]
    sc = StepConfig(model="lv", family="am", order=2, h=0.1, seed=seed, obs_idx=(0, 1), sigma=0.05)
    ens = O.init_uniform("lv", n, seed, **prob.prior)
    tp = 0.0
    for j in range(1, T + 1):
        trace_o, _ = O.pf_step(sc, ens, prob.ys[j - 1], j, tp, prob.times[j - 1])
        assert _rel(np.array(rows[j - 1]), trace_o) < REL_TRACE, j
        tp = prob.times[j - 1]


# ---------------------------------------------------------------- sharding
@pytest.mark.parametrize("world,pull", [(2, False), (4, False), (2, True), (4, True)])
def test_sharded_shards_reproduce_single_handle_bitwise(world, pull):
    """R shards (one GPU, LocalComm: phases strictly sequential, no kernel
    waits on another shard) reproduce the single-handle run bit for bit: the
    keyed streams use global slots, the LSE / moment partials are combined in
    the single-handle order, and the CDF is exact. pull: the migration as the
    peer-memory pull (k_pull reading the other shards' tables and records
    through a peer table of their device pointers; the multi-rank path of the
    native step's NVLink migration) instead of the counted exchange."""
    from paper_1411_1702_b200 import problems
    from paper_1411_1702_b200.sampler import GpuSampler
    from paper_1411_1702_b200.sharded import GpuShard, LocalComm, ShardedFilter
    n, T = 1 << 16, 4
    prob = problems.lotka_volterra(particles=n, T=T, seed=17)
    single = GpuSampler("lv", prob.cfg, prob.obs)
    single.initialize_uniform(**prob.prior)
    shards = [GpuShard("lv", prob.cfg, prob.obs, r, world) for r in range(world)]
    if pull:
        for s in shards:
            s.attach_peers_local(shards)
    f = ShardedFilter(shards, LocalComm(world), pull=pull)
    f.initialize_uniform(**prob.prior)
    e1, e2 = single.get_ensemble(), f.get_ensemble()
    assert np.array_equal(e1.states, e2.states) and np.array_equal(e1.params_u, e2.params_u)
    assert np.array_equal(e1.mean_u, e2.mean_u) and np.array_equal(e1.cov_u, e2.cov_u)
    tp = 0.0
    for j in range(1, T + 1):
        t1 = prob.times[j - 1]
        r1 = single.pf_step(prob.ys[j - 1], j, tp, t1)
        r2 = f.pf_step(prob.ys[j - 1], j, tp, t1, 0.1)
        a1, _, _ = single.step_diagnostics()
        assert np.array_equal(a1, f.ancestors()), f"step {j}: ancestors"
        for a, b in ((r1.theta_mean, r2.theta_mean), (r1.theta_var, r2.theta_var),
                     (r1.state_mean, r2.state_mean), ([r1.ess], [r2.ess])):
            assert np.array_equal(np.asarray(a), np.asarray(b)), f"step {j}: trace"
        tp = t1
    e1, e2 = single.get_ensemble(), f.get_ensemble()
    for name in ("states", "params_u", "logw", "mean_u", "cov_u"):
        assert np.array_equal(getattr(e1, name), getattr(e2, name)), name
    single.close()
    for s in shards:
        s.close()


def test_sharded_metabolic_adaptive_bitwise():
    """Sharding with the reference's own model and the adaptive integrator:
    2 shards (LocalComm, one GPU) == the single handle, bit for bit."""
    from paper_1411_1702_b200.sampler import GpuSampler, ObservationModel, PfConfig
    from paper_1411_1702_b200.sharded import GpuShard, LocalComm, ShardedFilter
    n = 1 << 15
    cfg = PfConfig(particles=n, shrink_a=0.98, seed=4, adaptive=True, rtol=1e-4)
    obs = ObservationModel([0, 1, 2], 0.1)
    prior = dict(th_mu=list(np.log([1.5, 0.7, 1.5, 0.5])), th_sigma=[0.5] * 4, x_mean=[1.0] * 3,
                 x_std=[0.25] * 3, x_clamp=[1, 1, 1])
    single = GpuSampler("metabolic", cfg, obs)
    single.initialize_gaussian(**prior)
    shards = [GpuShard("metabolic", cfg, obs, r, 2) for r in range(2)]
    f = ShardedFilter(shards, LocalComm(2))
    f.initialize_gaussian(**prior)
    rng = np.random.default_rng(2)
    tp = 1.6
    for j in range(1, 5):
        y = np.array([1.0, 1.2, 1.1]) + 0.1 * rng.standard_normal(3)
        r1 = single.pf_step(y, j, tp, tp + 0.2)
        r2 = f.pf_step(y, j, tp, tp + 0.2, 0.05)
        assert np.array_equal(single.step_diagnostics()[0], f.ancestors()), j
        for a, b in ((r1.theta_mean, r2.theta_mean), (r1.theta_var, r2.theta_var), ([r1.ess], [r2.ess])):
            assert np.array_equal(np.asarray(a), np.asarray(b)), j
        tp += 0.2
    e1, e2 = single.get_ensemble(), f.get_ensemble()
    for name in ("states", "params_u", "logw", "mean_u", "cov_u"):
        assert np.array_equal(getattr(e1, name), getattr(e2, name)), name
    single.close()
    for s in shards:
        s.close()


def test_sharded_torchcomm_nccl_world1_bitwise():
    """The multi-GPU orchestration path as bench.py --gpus N runs it (GpuShard +
    TorchComm over NCCL, collectives on the shard's stream), at world size 1 on
    this one GPU: every collective / exchange code path executes and the run
    equals the single handle bit for bit."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_1411_1702_b200 import problems
    from paper_1411_1702_b200.sampler import GpuSampler
    from paper_1411_1702_b200.sharded import GpuShard, ShardedFilter, TorchComm
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda:0"))
    try:
        n, T = 1 << 15, 4
        prob = problems.lotka_volterra(particles=n, T=T, seed=19)
        single = GpuSampler("lv", prob.cfg, prob.obs)
        single.initialize_uniform(**prob.prior)
        shard = GpuShard("lv", prob.cfg, prob.obs, 0, 1)
        f = ShardedFilter([shard], TorchComm())
        f.initialize_uniform(**prob.prior)
        shard2 = GpuShard("lv", prob.cfg, prob.obs, 0, 1)   # the native NCCL step
        f2 = ShardedFilter([shard2], TorchComm())
        f2.initialize_uniform(**prob.prior)
        shard2.attach_nccl()
        shard3 = GpuShard("lv", prob.cfg, prob.obs, 0, 1)   # native, migration pulled over peer memory
        f3 = ShardedFilter([shard3], TorchComm())
        f3.initialize_uniform(**prob.prior)
        shard3.attach_nccl()
        assert shard3.attach_peers()
        tp = 0.0
        for j in range(1, T + 1):
            t1 = prob.times[j - 1]
            r1 = single.pf_step(prob.ys[j - 1], j, tp, t1)
            r2 = f.pf_step(prob.ys[j - 1], j, tp, t1, 0.1)
            r3 = f2.pf_step(prob.ys[j - 1], j, tp, t1, 0.1)
            r4 = f3.pf_step(prob.ys[j - 1], j, tp, t1, 0.1)
            assert np.array_equal(single.step_diagnostics()[0], f.ancestors()), j
            assert np.array_equal(single.step_diagnostics()[0], f2.ancestors()), j
            assert np.array_equal(single.step_diagnostics()[0], f3.ancestors()), j
            assert np.array_equal(r1.theta_mean, r4.theta_mean) and r1.ess == r4.ess, j
            assert np.array_equal(r1.theta_mean, r2.theta_mean) and r1.ess == r2.ess, j
            assert np.array_equal(r1.theta_mean, r3.theta_mean) and r1.ess == r3.ess, j
            tp = t1
        e1, e2, e3, e4 = single.get_ensemble(), f.get_ensemble(), f2.get_ensemble(), f3.get_ensemble()
        for name in ("states", "params_u", "logw", "mean_u", "cov_u"):
            assert np.array_equal(getattr(e1, name), getattr(e2, name)), name
            assert np.array_equal(getattr(e1, name), getattr(e3, name)), name
            assert np.array_equal(getattr(e1, name), getattr(e4, name)), name
        single.close()
        shard.close()
        shard2.close()
        shard3.close()
    finally:
        dist.destroy_process_group()


def test_scan_modes_give_the_same_filter_bitwise():
    """The single-pass exact scan (decoupled look-back) and the two-pass form
    (records + resolver, CDF pass) give the same ancestors, ensemble and trace,
    bit for bit, over free-running steps (2^18 + a ragged tail: 129 tiles)."""
    from paper_1411_1702_b200 import problems
    n, steps = (1 << 18) + 333, 8
    prob = problems.lotka_volterra(particles=n, T=steps, seed=9)
    sc = StepConfig(model="lv", family="am", order=2, h=0.1, seed=9, obs_idx=(0, 1), sigma=0.05)
    out = {}
    for mode in SCAN_MODES:
        gpu = _sampler(sc, n)
        gpu.set_scan_mode(mode)
        gpu.initialize_uniform(**prob.prior)
        tp, rows, ancs = 0.0, [], []
        for j in range(1, steps + 1):
            t1 = prob.times[j - 1]
            row = gpu.pf_step(prob.ys[j - 1], j, tp, t1)
            rows.append(np.concatenate([row.theta_mean, row.theta_var, row.state_mean, [row.ess]]))
            ancs.append(gpu.step_diagnostics()[0].copy())
            tp = t1
        e = gpu.get_ensemble()
        out[mode] = (np.array(rows), np.array(ancs), e.states.copy(), e.params_u.copy(), e.logw.copy())
        gpu.close()
    for a, b in zip(out["fused"], out["two_pass"]):
        assert np.array_equal(a, b)


def test_free_running_full_size_lv():
    """BASELINE config 2 size (N = 2^20): 10 free-running steps, ancestors
    bit-exact against the oracle and the trace within 1e-8."""
    from paper_1411_1702_b200 import problems
    n, steps = 1 << 20, 10
    prob = problems.lotka_volterra(particles=n, T=steps, seed=1)
    sc = StepConfig(model="lv", family="am", order=2, h=0.1, seed=1, obs_idx=(0, 1), sigma=0.05)
    ens = O.init_uniform("lv", n, 1, **prob.prior)
    gpu = _sampler(sc, n)
    gpu.set_ensemble(_to_gpu_ens(ens))
    tp = 0.0
    for j in range(1, steps + 1):
        t1 = prob.times[j - 1]
        row = gpu.pf_step(prob.ys[j - 1], j, tp, t1)
        trace_o, dg = O.pf_step(sc, ens, prob.ys[j - 1], j, tp, t1, diag=True)
        anc_g, _, _ = gpu.step_diagnostics()
        mism = np.count_nonzero(anc_g.astype(np.int64) != dg["ancestors"])
        assert mism == 0, f"step {j}: {mism} ancestors differ"
        tr = np.concatenate([row.theta_mean, row.theta_var, row.state_mean, [row.ess]])
        assert _rel(tr, trace_o) < REL_TRACE, j
        tp = t1
    gpu.close()


@pytest.mark.parametrize("n,sigmas", [(1 << 16, (0.1, 1.0, 4.0)), ((1 << 22) + 4097 * 3 + 5, (1.0,))])
def test_c5_resample_iteration_matches_oracle(n, sigmas):
    """BASELINE config 5 iteration on 64-byte records: LSE, weighted 2x2
    covariance, exact multinomial resampling and the gather, vs the oracle's
    fitness_weights / weighted_mean_cov / resample_multinomial. The second
    case is ragged and uses the 4096-element tiles."""
    from paper_1411_1702_b200.sampler import Ensemble, GpuSampler, ObservationModel, PfConfig
    rng = np.random.default_rng(3)
    for sigma in sigmas:
        s = GpuSampler("payload64", PfConfig(particles=n, seed=77), ObservationModel([0], 1.0))
        states = rng.standard_normal((n, 6))
        params = rng.standard_normal((n, 2))
        s.set_ensemble(Ensemble(states, params, np.zeros(n), np.zeros(2), np.eye(2)))
        s.c5_set_logweights(sigma, 5)
        lw = s.get_ensemble().logw.copy()
        s.c5_iteration(1)
        s.synchronize()
        anc, _, _ = s.step_diagnostics()
        g = O.fitness(lw, np.zeros(n))
        want = O.resample(g, 77, 1)
        anc = anc.astype(np.int64)
        # The reference's lse is a sequential sum (relative error up to ~n eps);
        # ours is a tree. Every g therefore moves by that much and a slot whose
        # uniform sits that close to a CDF edge may legitimately flip: such
        # classified near-ties are the only mismatches allowed.
        bad = np.nonzero(anc != want)[0]
        if len(bad):
            cdf = np.cumsum(g)
            cdf[-1] = max(cdf[-1], 1.0)
            tol = 4.0 * n * 2.0 ** -53
            for b in bad:
                u = O.draws(77, 1, int(b), 3, 1, 1)[0]
                edge = cdf[min(anc[b], want[b])]
                assert abs(u - edge) <= tol * edge, (sigma, b, u, edge)
            assert len(bad) <= 8, (sigma, len(bad))
        # exactness of the device CDF itself: the oracle's own g injected
        a2, cdf2 = s.resample_from_g(g, 1, with_cdf=True)
        assert np.array_equal(a2.astype(np.int64), want), sigma
        cdf_o = np.cumsum(g)
        cdf_o[-1] = max(cdf_o[-1], 1.0)
        assert np.array_equal(cdf2, cdf_o), sigma
        e = s.get_ensemble()
        assert np.array_equal(e.states, states[anc]) and np.array_equal(e.params_u, params[anc])
        mean, cov = O.weighted_mean_cov(params, g)
        np.testing.assert_allclose(e.mean_u, mean, rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(e.cov_u, cov, rtol=1e-8, atol=1e-13)
        s.close()


@pytest.mark.parametrize("n,cap", [(1 << 16, 0), ((1 << 22) + 4097 * 3 + 5, 0), ((1 << 20) + 77, 0),
                                   (1 << 16, 256), (3 * 4096 + 11, 512)])
def test_c5_bucketed_search_is_the_slot_order_search(n, cap):
    """The bucketed ancestor search (uniforms partitioned by value, served in
    bucket order) gives every slot the slot-order search's ancestor and record,
    bit for bit; cap > 0 forces a tiny bucket capacity so most items take the
    spill list."""
    from paper_1411_1702_b200.sampler import Ensemble, GpuSampler, ObservationModel, PfConfig
    rng = np.random.default_rng(11)
    states = rng.standard_normal((n, 6))
    params = rng.standard_normal((n, 2))
    out = {}
    for mode in ("guide", "bucketed", "split"):
        s = GpuSampler("payload64", PfConfig(particles=n, seed=78), ObservationModel([0], 1.0))
        s.c5_set_search(mode, debug_bucket_cap=cap if mode == "bucketed" else 0)
        s.set_ensemble(Ensemble(states, params, np.zeros(n), np.zeros(2), np.eye(2)))
        s.c5_set_logweights(2.0, 9)
        res = []
        for it in range(1, 4):  # chained iterations: the second and third resample the first's output
            s.c5_iteration(it)
            s.synchronize()
            anc, _, _ = s.step_diagnostics()
            e = s.get_ensemble()
            res.append((anc.copy(), e.states.copy(), e.params_u.copy(), e.mean_u.copy(), e.cov_u.copy()))
        out[mode] = res
        s.close()
    for other in ("bucketed", "split"):
        for a, b in zip(out["guide"], out[other]):
            for x, y in zip(a, b):
                assert np.array_equal(x, y), other


@pytest.mark.parametrize("n", [1 << 16, (1 << 22) + 4097 * 3 + 5])
def test_c5_gather_moments_are_the_stats_pass_moments(n):
    """SPLIT search: from the second iteration on the stats pass takes each
    tile's weighted-moment sums from the previous iteration's gather
    (k_c5_gather_moments) instead of reading theta again. Same tiles, thread
    layout and trees: the mean, covariance, ancestors and records are bitwise
    those of the pass that reads theta itself, also after the log-weights change."""
    from paper_1411_1702_b200.sampler import Ensemble, GpuSampler, ObservationModel, PfConfig
    rng = np.random.default_rng(8)
    states = rng.standard_normal((n, 6))
    params = rng.standard_normal((n, 2))
    out = {}
    for fuse in (True, False):
        s = GpuSampler("payload64", PfConfig(particles=n, seed=12), ObservationModel([0], 1.0))
        s.c5_set_search("split")
        s.c5_fuse_moments(fuse)
        s.set_ensemble(Ensemble(states, params, np.zeros(n), np.zeros(2), np.eye(2)))
        rows = []
        for sigma, key in ((1.0, 3), (4.0, 9)):
            s.c5_set_logweights(sigma, key)
            for it in range(3):
                s.c5_iteration(10 * key + it)
                s.synchronize()
                e = s.get_ensemble()
                rows.append((e.mean_u.copy(), e.cov_u.copy(), s.step_diagnostics()[0].copy()))
        e = s.get_ensemble()
        out[fuse] = (rows, e.states.copy(), e.params_u.copy())
        s.close()
    for (m1, c1, a1), (m0, c0, a0) in zip(out[True][0], out[False][0]):
        assert np.array_equal(m1, m0) and np.array_equal(c1, c0) and np.array_equal(a1, a0)
    assert np.array_equal(out[True][1], out[False][1]) and np.array_equal(out[True][2], out[False][2])


def test_c5_bucket_spill_overflow_raises():
    """More items than bucket capacity + spill list: an internal error at the
    next synchronize, not a silent partial gather."""
    from paper_1411_1702_b200.sampler import Ensemble, GpuSampler, ObservationModel, PfConfig
    n = 1 << 17
    s = GpuSampler("payload64", PfConfig(particles=n, seed=78), ObservationModel([0], 1.0))
    s.c5_set_search("bucketed", debug_bucket_cap=256)
    s.set_ensemble(Ensemble(np.zeros((n, 6)), np.zeros((n, 2)), np.zeros(n), np.zeros(2), np.eye(2)))
    s.c5_set_logweights(1.0, 9)
    s.c5_iteration(1)
    with pytest.raises(Exception, match="internal"):
        s.synchronize()
    s.close()


# ---------------------------------------------------------------- error paths of chol_psd / weights
def _err_sampler_and_ens(n=4096, seed=3):
    sc = StepConfig(model="lv", family="am", order=2, h=0.1, a=0.98, seed=seed, obs_idx=(0, 1), sigma=0.05)
    ens = O.init_uniform("lv", n, seed, [0.5, 0.5], [1.5, 1.5], [0.5, 0.5], [1.5, 1.5])
    return sc, ens, _sampler(sc, n)


def test_chol_jitter_rung_above_zero_matches_oracle():
    """cov_u slightly indefinite: chol_psd's ladder (linalg.cpp:486-498)
    fails the first rungs and succeeds with a positive jitter (1e-6 tr/p
    here); the proliferation uses that jittered factor on both sides."""
    sc, ens, gpu = _err_sampler_and_ens()
    c = 1e-2
    ens.cov_u = np.array([[c, c * (1 + 1e-7)], [c * (1 + 1e-7), c]])
    L, jit = O.chol_psd(ens.cov_u)
    assert any(jit == r * c for r in (1e-12, 1e-10, 1e-8, 1e-6, 1e-4)) and jit > 0  # a rung above 0
    gpu.set_ensemble(_to_gpu_ens(ens))
    row = gpu.pf_step([1.1, 0.9], 1, 0.0, 0.1)
    trace_o, dg = O.pf_step(sc, ens, [1.1, 0.9], 1, 0.0, 0.1, diag=True)
    _compare_step(gpu, ens, trace_o, dg, row)
    gpu.close()


@pytest.mark.parametrize("case", ["chol_failure", "weights_sum", "asymmetric_cov"])
def test_injected_ensemble_errors_match_reference(case):
    """An ensemble the reference's pf_step rejects: a covariance no rung of
    the jitter ladder can factor (NUMERICAL "chol_psd: degenerate covariance",
    linalg.cpp:499), weights that do not sum to 1 (CONFIG, the Kahan gate of
    weighted_mean_cov, linalg.cpp:395-409) and an asymmetric covariance
    (chol_psd's symmetry check, std::invalid_argument -> INTERNAL,
    linalg.cpp:474-480). Same status family and message on the GPU as in the
    C oracle and (when built) the live reference, at the same step."""
    from oracle_ctypes import REF_SO, OracleError, Reference
    from paper_1411_1702_b200.sampler import ConfigError, NumericalError, PfsmcError
    sc, ens, gpu = _err_sampler_and_ens()
    if case == "chol_failure":
        ens.cov_u = np.array([[1.0, 2.0], [2.0, 1.0]])
        want_cls, code, msg = NumericalError, 3, "chol_psd: degenerate covariance"
    elif case == "weights_sum":
        ens.logw = ens.logw + 1e-9
        want_cls, code, msg = ConfigError, 2, "weighted_mean_cov: weights must sum to 1"
    else:
        ens.cov_u = ens.cov_u.copy()
        ens.cov_u[0, 1] += 1e-9
        want_cls, code, msg = PfsmcError, 1, "chol_psd: matrix must be symmetric"
    gpu.set_ensemble(_to_gpu_ens(ens))
    with pytest.raises(want_cls) as e:
        gpu.pf_step([1.1, 0.9], 1, 0.0, 0.1)
    assert msg in str(e.value)
    assert type(e.value) is want_cls or want_cls is PfsmcError
    checkers = [O] + ([Reference()] if os.path.exists(REF_SO) else [])
    for chk in checkers:
        with pytest.raises(OracleError) as eo:
            chk.pf_step(sc, ens.copy(), [1.1, 0.9], 1, 0.0, 0.1)
        assert msg in str(eo.value), (chk, eo.value)
        if chk is not O:
            assert eo.value.code == code, eo.value
    gpu.close()
