"""Pins the CPU oracle (oracle/pfsmc_oracle.c) before anything is checked
against it: golden vectors from the reference's own tests, fixtures produced
by the unmodified reference (tests/golden/make_golden.py), the reference's
scripted one-step trace (test_filter.cpp:363-453) and, where the reference
build is present, live bitwise comparison with it. CPU only."""
import json
import math
import os

import numpy as np
import pytest

from oracle_ctypes import METABOLIC_DEFAULTS, REF_SO, Oracle, OracleError, Reference, StepConfig, set_advdiff_grid

GOLD = os.path.join(os.path.dirname(__file__), "golden")
O = Oracle()
HAVE_REF = os.path.exists(REF_SO)


def test_philox_known_answers():
    # rng.cpp:28-41 against tests/data/philox_vectors.csv (test_rng.cpp:16-44)
    kats = json.load(open(os.path.join(GOLD, "philox_vectors.json")))["vectors"]
    assert len(kats) == 4
    for k in kats:
        out = O.philox([int(x, 16) for x in k["ctr"]], [int(x, 16) for x in k["key"]])
        assert [f"{int(x):016x}" for x in out] == k["out"]


def test_streams_match_reference_draws():
    st = json.load(open(os.path.join(GOLD, "rng_streams.json")))["streams"]
    for key, v in st.items():
        seed, j, n, purpose = map(int, key.split("_"))
        assert [f"{int(x):016x}" for x in O.draws(seed, j, n, purpose, 0, 9)] == v["u64"]
        assert [float.hex(float(x)) for x in O.draws(seed, j, n, purpose, 1, 9)] == v["uniform"]
        assert [float.hex(float(x)) for x in O.draws(seed, j, n, purpose, 2, 9)] == v["normal"]


def test_stream_purity_and_ranges():
    # test_rng.cpp:46-70
    a = O.draws(123, 5, 17, 2, 0, 100)
    assert np.array_equal(a, O.draws(123, 5, 17, 2, 0, 100))
    for other in [(123, 5, 17, 1), (123, 5, 18, 2), (124, 5, 17, 2), (123, 6, 17, 2)]:
        assert O.draws(*other, 0, 1)[0] != a[0]
    u = O.draws(7, 0, 0, 0, 1, 10000)
    assert u.min() >= 0.0 and u.max() < 1.0
    z = O.draws(42, 3, 0, 1, 2, 200000)
    assert abs(z.mean()) < 0.01 and abs(z.var() - 1.0) < 0.02


def _golden_cases():
    return sorted(f[3:-4] for f in os.listdir(GOLD) if f.startswith("pf_") and f.endswith(".npz"))


def _ens_from(d, prefix):
    from oracle_ctypes import Ensemble
    return Ensemble(d[f"{prefix}states"].copy(), d[f"{prefix}params_u"].copy(), d[f"{prefix}logw"].copy(),
                    d[f"{prefix}mean_u"].copy(), d[f"{prefix}cov_u"].copy())


@pytest.mark.parametrize("case", _golden_cases())
def test_oracle_replays_reference_bitwise(case):
    """Every field of every step equals the unmodified reference bit for bit."""
    d = np.load(os.path.join(GOLD, f"pf_{case}.npz"))
    sc = StepConfig(**json.loads(str(d["config"])))
    if sc.model == "advdiff":
        set_advdiff_grid(int(d["model_consts"][0]), O)
    try:
        ens = _ens_from(d, "init_")
        for j, (t0, t1, h) in enumerate(d["steps"], 1):
            sc.h = float(h)
            trace, dg = O.pf_step(sc, ens, d["ys"][j - 1], j, float(t0), float(t1), diag=True)
            assert np.array_equal(dg["ancestors"], d[f"s{j}_anc"])
            assert np.array_equal(dg["g"], d[f"s{j}_g"])
            assert np.array_equal(dg["loglik_bar"], d[f"s{j}_llbar"])
            assert np.array_equal(trace, d[f"s{j}_trace"])
            for f in ("states", "params_u", "logw", "mean_u", "cov_u"):
                assert np.array_equal(getattr(ens, f), d[f"s{j}_{f}"]), (case, j, f)
    finally:
        O.set_model_consts(METABOLIC_DEFAULTS)


def test_oracle_resample_matches_reference_fixture():
    d = np.load(os.path.join(GOLD, "resample.npz"))
    for k in [x[:-2] for x in d.files if x.endswith("_g")]:
        assert np.array_equal(O.resample(d[f"{k}_g"], 99, 4), d[f"{k}_anc"]), k


def test_resample_edge_cases():
    # test_filter.cpp:179-229: one-hot, determinism, chi-square, last-bin guard
    onehot = np.zeros(8)
    onehot[3] = 1.0
    assert np.all(O.resample(onehot, 1, 1) == 3)
    g = np.full(100, 0.01)
    assert np.array_equal(O.resample(g, 7, 4), O.resample(g, 7, 4))
    assert not np.array_equal(O.resample(g, 7, 4), O.resample(g, 8, 4))
    n = 100000
    draws = O.resample(np.full(n, 1.0 / n), 42, 1)
    counts = np.bincount(draws // (n // 10), minlength=10)
    chi2 = ((counts - n / 10) ** 2 / (n / 10)).sum()
    assert chi2 < 27.877
    short = np.full(10, 0.09)  # sums to 0.9: draws above land on the last bin
    anc = O.resample(short, 5, 2)
    assert anc.max() <= 9 and np.any(anc == 9)


def test_scripted_three_particle_step():
    """Restates the reference's brute-force trace (test_filter.cpp:363-453):
    x' = -theta x, BDF1, one internal step, closed forms + keyed streams."""
    seed, a, h = 31415, 0.95, 0.5
    y = 1.2
    th_u = np.zeros(3)
    x0 = np.zeros(3)
    for i in range(3):
        z = O.draws(seed, 0, i, 0, 2, 2)
        th_u[i] = math.log(0.8) + 0.4 * z[0]
        x0[i] = 2.0 + 0.1 * z[1]
    mean_u = th_u.sum() / 3.0
    c0 = sum((v - mean_u) ** 2 / 3.0 for v in th_u)

    def loglik(x):
        return -0.5 * math.log(2.0 * math.pi * 0.25) - (y - x) ** 2 / (2.0 * 0.25)

    th_bar = a * th_u + (1 - a) * mean_u
    xbar = x0 / (1.0 + h * np.exp(th_bar))
    llb = np.array([loglik(v) for v in xbar])
    g = np.exp(llb) / 3.0
    g /= g.sum()
    anc = []
    for i in range(3):
        u = O.draws(seed, 1, i, 3, 1, 1)[0]
        anc.append(0 if u < g[0] else (1 if u < g[0] + g[1] else 2))
    th_new = np.zeros(3)
    x_new = np.zeros(3)
    ll_new = np.zeros(3)
    for i in range(3):
        th_new[i] = th_bar[anc[i]] + math.sqrt(1 - a * a) * math.sqrt(c0) * O.draws(seed, 1, i, 1, 2, 1)[0]
        tn = math.exp(th_new[i])
        corr = x0[anc[i]] / (1.0 + h * tn)
        pred = x0[anc[i]] * (1.0 - h * tn)
        gamma = 0.25 * (corr - pred) ** 2
        x_new[i] = corr + math.sqrt(gamma) * O.draws(seed, 1, i, 2, 2, 1)[0]
        ll_new[i] = loglik(x_new[i])
    lw = ll_new - llb[anc]
    w = np.exp(lw - (lw.max() + math.log(np.exp(lw - lw.max()).sum())))

    ens = O.init_gaussian("decay", 3, seed, [math.log(0.8)], [0.4], [2.0], [0.1], [0])
    sc = StepConfig(model="decay", family="bdf", order=1, h=h, a=a, seed=seed, obs_idx=(0,), sigma=0.5)
    trace, dg = O.pf_step(sc, ens, [y], 1, 0.0, 0.5, diag=True)
    assert list(dg["ancestors"]) == anc
    np.testing.assert_allclose(ens.params_u[:, 0], th_new, rtol=1e-12)
    np.testing.assert_allclose(ens.states[:, 0], x_new, rtol=1e-9)
    np.testing.assert_allclose(np.exp(ens.logw), w, rtol=1e-9)
    np.testing.assert_allclose(trace[0], math.exp((w * th_new).sum()), rtol=1e-10)
    np.testing.assert_allclose(trace[-1], 1.0 / (w * w).sum(), rtol=1e-9)


def test_block_functions_and_errors():
    g = O.fitness(np.full(2, -math.log(2)), [0.0, -math.inf])
    assert g[0] == 1.0 and g[1] == 0.0
    with pytest.raises(OracleError) as e:
        O.fitness(np.full(2, -math.log(2)), [-math.inf, -math.inf])
    assert e.value.code == 3
    # chol_psd jitter ladder: exactly singular PSD is accepted, negative-definite fails
    L, jit = O.chol_psd(np.array([[1.0, 1.0], [1.0, 1.0]]))
    assert jit == 0.0 and L[1, 1] == 0.0
    with pytest.raises(OracleError):
        O.chol_psd(np.array([[1.0, 0.0], [0.0, -1.0]]))
    m, c = O.weighted_mean_cov(np.array([[0.0], [1.0], [2.0], [5.0]]), np.full(4, 0.25))
    assert m[0] == 2.0 and abs(c[0, 0] - 3.5) < 1e-15


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("family,order,h", [("ab", 1, 0.1), ("ab", 2, 0.05), ("am", 2, 0.1), ("am", 3, 0.025),
                                            ("bdf", 2, 0.05), ("bdf", 3, 0.02)])
def test_oracle_matches_live_reference(family, order, h):
    R = Reference()
    sc = StepConfig(model="lv", family=family, order=order, h=h, seed=17)
    e = O.init_uniform("lv", 300, 17, [0.5, 0.5], [1.5, 1.5], [0.5, 0.5], [1.5, 1.5])
    e2 = e.copy()
    rng = np.random.default_rng(1)
    tp = 0.0
    for j in range(1, 5):
        y = np.array([1.2, 0.9]) + 0.1 * rng.standard_normal(2)
        t1, _ = O.pf_step(sc, e, y, j, tp, tp + 0.1)
        t2 = R.pf_step(sc, e2, y, j, tp, tp + 0.1)
        tp += 0.1
        assert np.array_equal(t1, t2)
        assert np.array_equal(e.states, e2.states) and np.array_equal(e.logw, e2.logw)


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("family,order,consts", [("bdf", 2, None), ("am", 3, None), ("ab", 2, None),
                                                 ("bdf", 3, (0.7, 0.5, 1.2, 3.0, 1.9, 0.6))])
def test_oracle_matches_live_reference_metabolic(family, order, consts):
    """The reference's own MetabolicModel (time-dependent input flux) through
    the reference's initialize (Gaussian prior, clamped x0) and pf_step; the
    steps straddle the input switch-on at t0_input so both branches of
    input_phi (models.cpp:37-42) run, with m = 4 sub-steps per interval."""
    R = Reference()
    k = consts or (1.0, 1.0, 1.0, 5.0, 2.0, 1.0)
    O.set_model_consts(k)
    R.set_model_consts(k)
    try:
        sc = StepConfig(model="metabolic", family=family, order=order, h=0.05, seed=5, obs_idx=(0, 1, 2),
                        sigma=0.1)
        mu = np.log([1.5, 0.7, 1.5, 0.5])
        e = O.init_gaussian("metabolic", 400, 5, mu, [0.5] * 4, [1.0] * 3, [0.25] * 3, [1, 1, 1])
        e2 = R.init_gaussian(sc, 400, mu, [0.5] * 4, [1.0] * 3, [0.25] * 3, [1, 1, 1])
        assert np.array_equal(e.states, e2.states) and np.array_equal(e.params_u, e2.params_u)
        rng = np.random.default_rng(3)
        tp = 1.6
        for j in range(1, 6):
            y = np.array([1.0, 1.2, 1.1]) + 0.1 * rng.standard_normal(3)
            t1, _ = O.pf_step(sc, e, y, j, tp, tp + 0.2)
            t2 = R.pf_step(sc, e2, y, j, tp, tp + 0.2)
            tp += 0.2
            assert np.array_equal(t1, t2), j
            assert np.array_equal(e.states, e2.states) and np.array_equal(e.logw, e2.logw)
    finally:
        O.set_model_consts((1.0, 1.0, 1.0, 5.0, 2.0, 1.0))
        R.set_model_consts((1.0, 1.0, 1.0, 5.0, 2.0, 1.0))


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("model,rtol", [("metabolic", 1e-3), ("metabolic", 1e-5), ("lv", 1e-4),
                                        ("robertson", 1e-3)])
def test_oracle_matches_live_reference_adaptive(model, rtol):
    """Variable-step BDF(1,2) (adaptive_bdf_interval, lmm.cpp:894-1019) through
    pf_step: oracle == unmodified reference, every field, bitwise."""
    R = Reference()
    rng = np.random.default_rng(9)
    if model == "metabolic":
        sc = StepConfig(model=model, family="bdf", order=2, seed=6, obs_idx=(0, 1, 2), sigma=0.1,
                        adaptive=True, rtol=rtol)
        mu = np.log([1.5, 0.7, 1.5, 0.5])
        e = O.init_gaussian(model, 300, 6, mu, [0.5] * 4, [1.0] * 3, [0.25] * 3, [1, 1, 1])
        ys = [np.array([1.0, 1.2, 1.1]) + 0.1 * rng.standard_normal(3) for _ in range(4)]
        ts = [1.6 + 0.2 * k for k in range(5)]
    elif model == "lv":
        sc = StepConfig(model=model, family="bdf", order=2, seed=6, adaptive=True, rtol=rtol)
        e = O.init_uniform("lv", 300, 6, [0.5, 0.5], [1.5, 1.5], [0.5, 0.5], [1.5, 1.5])
        ys = [np.array([1.2, 0.9]) + 0.05 * rng.standard_normal(2) for _ in range(4)]
        ts = [0.1 * k for k in range(5)]
    else:
        sc = StepConfig(model=model, family="bdf", order=2, a=0.99, seed=6, obs_idx=(0, 2), sigma=0.02,
                        newton_max_iter=4, likelihood="gaussian", adaptive=True, rtol=rtol)
        e = R.init_gaussian(sc, 200, np.log([0.04, 3e7, 1e4]) + 0.5, [1, 1, 1], [1, 0, 0], [0, 0, 0], [0, 0, 0])
        ts = [0.0] + list(np.logspace(-4, 3, 400)[:4])
        ys = [np.array([1 - 0.04 * t, 0.04 * t * 1e-3]) + 1e-3 * rng.standard_normal(2) for t in ts[1:]]
    e2 = e.copy()
    for j in range(1, len(ts)):
        t1, _ = O.pf_step(sc, e, ys[j - 1], j, ts[j - 1], ts[j])
        t2 = R.pf_step(sc, e2, ys[j - 1], j, ts[j - 1], ts[j])
        assert np.array_equal(t1, t2), j
        assert np.array_equal(e.states, e2.states) and np.array_equal(e.logw, e2.logw)
        assert np.array_equal(e.params_u, e2.params_u)


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (needs /root/reference)")
def test_degeneracy_error_parity():
    """Both raise NUMERICAL at the same step (total degeneracy)."""
    R = Reference()
    sc = StepConfig(model="lv", family="am", order=1, h=0.1, seed=2)
    e = O.init_uniform("lv", 64, 2, [0.5, 0.5], [1.5, 1.5], [0.5, 0.5], [1.5, 1.5])
    far = np.array([1e200, 1e200])  # r^2 overflows: every log-lik is -inf
    with pytest.raises(OracleError) as a:
        O.pf_step(sc, e.copy(), far, 1, 0.0, 0.1)
    with pytest.raises(OracleError) as b:
        R.pf_step(sc, e.copy(), far, 1, 0.0, 0.1)
    assert a.value.code == b.value.code == 3
