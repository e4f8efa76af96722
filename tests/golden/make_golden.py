"""Regenerates the committed golden fixtures from the UNMODIFIED reference
(oracle/_ref/libpfsmc_ref.so, built from /root/reference by oracle/Makefile)
and from the reference's own test data. Run here (the dev container), not on
the GPU box: /root/reference does not exist there.

  python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_ctypes import Oracle, Reference, StepConfig, set_advdiff_grid  # noqa: E402

REF_KAT = "/root/reference/proj/tests/data/philox_vectors.csv"


def philox_kats():
    rows = []
    for line in open(REF_KAT):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.strip().split(",")]
        rows.append({"ctr": [f"{x:016x}" for x in v[:4]], "key": [f"{x:016x}" for x in v[4:6]],
                     "out": [f"{x:016x}" for x in v[6:10]]})
    json.dump({"source": "reference tests/data/philox_vectors.csv (Philox4x64-10 KATs)",
               "vectors": rows}, open(os.path.join(HERE, "philox_vectors.json"), "w"), indent=1)


def streams():
    R = Reference()
    out = {}
    for (seed, j, n, purpose) in [(123, 5, 17, 2), (42, 3, 0, 1), (7, 0, 0, 0), (31415, 1, 2, 3)]:
        out[f"{seed}_{j}_{n}_{purpose}"] = {
            "u64": [f"{x:016x}" for x in R.draws(seed, j, n, purpose, 0, 9)],
            "uniform": [float.hex(float(x)) for x in R.draws(seed, j, n, purpose, 1, 9)],
            "normal": [float.hex(float(x)) for x in R.draws(seed, j, n, purpose, 2, 9)]}
    json.dump({"source": "reference rng::RngStream via oracle/_ref", "streams": out},
              open(os.path.join(HERE, "rng_streams.json"), "w"), indent=1)


CASES = {
    # name: (StepConfig kwargs, n, init, steps (t_prev, t_obs, h), y rows)
    "lv_am2_m1": (dict(model="lv", family="am", order=2, h=0.1, a=0.98, seed=11, obs_idx=(0, 1), sigma=0.05),
                  96, "uniform_lv", [(0.1 * k, 0.1 * (k + 1), 0.1) for k in range(6)]),
    "lv_ab3_m4": (dict(model="lv", family="ab", order=3, h=0.025, a=0.98, seed=12, obs_idx=(0, 1), sigma=0.05),
                  64, "uniform_lv", [(0.1 * k, 0.1 * (k + 1), 0.025) for k in range(4)]),
    "lv_bdf3_m4": (dict(model="lv", family="bdf", order=3, h=0.025, a=0.98, seed=13, obs_idx=(0, 1), sigma=0.05),
                   64, "uniform_lv", [(0.1 * k, 0.1 * (k + 1), 0.025) for k in range(4)]),
    "chain_bdf3_m3": (dict(model="chain", family="bdf", order=3, h=0.1 / 3, a=0.98, seed=5, obs_idx=(0, 3, 7),
                           sigma=0.01), 48, "uniform_chain", [(0.1 * k, 0.1 * (k + 1), 0.1 / 3) for k in range(3)]),
    "robertson_bdf2_m2": (dict(model="robertson", family="bdf", order=2, a=0.99, seed=3, obs_idx=(0, 2),
                               sigma=0.02, newton_max_iter=4), 48, "gauss_rob", None),
    "decay_bdf1": (dict(model="decay", family="bdf", order=1, h=0.5, a=0.95, seed=31415, obs_idx=(0,), sigma=0.5),
                   3, "gauss_decay", [(0.0, 0.5, 0.5)]),
    # the reference's own MetabolicModel (default MetabolicConstants), across the input switch-on
    "metabolic_bdf2_m4": (dict(model="metabolic", family="bdf", order=2, h=0.05, a=0.98, seed=21,
                               obs_idx=(0, 1, 2), sigma=0.1), 80, "gauss_metabolic",
                          [(1.6 + 0.2 * k, 1.6 + 0.2 * (k + 1), 0.05) for k in range(5)]),
    # the reference's own AdvDiffModel (problem 2), grid n = 6 (d = 25) / 5 (d = 16): bench.cpp:249-277
    # priors, the plume x0 as a degenerate prior, sites drawn like generate_data (bench.cpp:327-341)
    "advdiff_bdf2_n6": (dict(model="advdiff", family="bdf", order=2, h=0.05, a=0.98, seed=17,
                             obs_idx=(3, 7, 11, 20, 24), sigma=0.05), 48, "gauss_advdiff_6",
                        [(float(k), float(k + 1), 0.05) for k in range(3)]),
    "advdiff_am3_n5": (dict(model="advdiff", family="am", order=3, h=0.1, a=0.98, seed=18,
                            obs_idx=(0, 5, 9, 14), sigma=0.05), 40, "gauss_advdiff_5",
                       [(float(k), float(k + 1), 0.1) for k in range(3)]),
    "advdiff_adaptive_n5": (dict(model="advdiff", family="bdf", order=2, a=0.98, seed=19,
                                 obs_idx=(1, 6, 12), sigma=0.05, adaptive=True, rtol=1e-3), 32,
                            "gauss_advdiff_5", [(float(k), float(k + 1), 1.0) for k in range(2)]),
}
# grid parameter of the advdiff cases (AdvDiffModel(n), model_consts[0])
CONSTS = {"advdiff_bdf2_n6": (6.0,), "advdiff_am3_n5": (5.0,), "advdiff_adaptive_n5": (5.0,)}
ADV_TRUTH = np.array([9.0, 4.0, 6.0, 2.5, -1.5])  # bench.cpp:251-255


def init_ens(kind, n, seed, O, R, sc):
    if kind == "uniform_lv":
        return O.init_uniform("lv", n, seed, [0.5, 0.5], [1.5, 1.5], [0.5, 0.5], [1.5, 1.5])
    if kind == "uniform_chain":
        th = np.array([2.0, 50.0, 5.0, 0.5])
        return O.init_uniform("chain", n, seed, 0.5 * th, 2 * th, [0] * 8, [0] * 8)
    if kind == "gauss_rob":
        return R.init_gaussian(sc, n, np.log([0.04, 3e7, 1e4]) + 0.5, [1, 1, 1], [1, 0, 0], [0, 0, 0], [0, 0, 0])
    if kind == "gauss_metabolic":  # bench.cpp:214-237 defaults
        return R.init_gaussian(sc, n, np.log([1.5, 0.7, 1.5, 0.5]), [0.5] * 4, [1.0] * 3, [0.25] * 3, [1, 1, 1])
    if kind.startswith("gauss_advdiff_"):  # bench.cpp:259-272
        g = int(kind.rsplit("_", 1)[1])
        x0 = plume(O, g)
        return R.init_gaussian(sc, n, [np.log(7.0), np.log(5.0), 4.0, 0.0, 0.0], [0.35, 0.35, 2.0, 2.0, 2.0],
                               x0, np.zeros_like(x0), np.zeros(len(x0), np.int32))
    if kind == "gauss_decay":
        return R.init_gaussian(sc, n, [np.log(0.8)], [0.4], [2.0], [0.1], [0])
    raise KeyError(kind)


def plume(O, g):
    import ctypes as C
    x0 = np.zeros((g - 1) ** 2)
    O.lib.or_gaussian_plume_ic(g, x0.ctypes.data_as(C.POINTER(C.c_double)))
    return x0


def pf_cases():
    O, R = Oracle(), Reference()
    rng = np.random.default_rng(2024)
    for name, (kw, n, init, steps) in CASES.items():
        sc = StepConfig(**kw)
        consts = CONSTS.get(name)
        if kw["model"] == "advdiff":
            set_advdiff_grid(int(consts[0]), O, R)
        if steps is None:  # log-spaced Robertson intervals, m = 2
            ts = np.logspace(-4, 3, 400)[:4]
            tp = np.concatenate([[0.0], ts[:-1]])
            steps = [(a, b, (b - a) / 2) for a, b in zip(tp, ts)]
        ens = init_ens(init, n, kw["seed"], O, R, sc)
        d = {"config": json.dumps(kw), "n": n}
        if consts:
            d["model_consts"] = np.array(consts)
        truth = plume(O, int(consts[0])) if kw["model"] == "advdiff" else None
        d["init_states"], d["init_params_u"], d["init_logw"] = ens.states.copy(), ens.params_u.copy(), ens.logw.copy()
        d["init_mean_u"], d["init_cov_u"] = ens.mean_u.copy(), ens.cov_u.copy()
        d["steps"] = np.array(steps)
        ys = []
        for j, (t0, t1, h) in enumerate(steps, 1):
            sc.h = h
            if kw["model"] == "lv":
                y = np.array([1.2, 0.9]) + 0.05 * rng.standard_normal(2)
            elif kw["model"] == "chain":
                y = np.array([0.09 * j, 0.001 * j, 0.0]) + 0.01 * rng.standard_normal(3)
            elif kw["model"] == "metabolic":
                y = np.array([1.0, 1.2, 1.1]) + 0.1 * rng.standard_normal(3)
            elif kw["model"] == "advdiff":  # truth path (fine BDF2) + N(0, sigma^2) at the sites
                truth = O.propagate("advdiff", ADV_TRUTH, truth, t0, t1, 0.01, "bdf", 2)[0]
                y = truth[list(kw["obs_idx"])] + kw["sigma"] * rng.standard_normal(len(kw["obs_idx"]))
            elif kw["model"] == "robertson":
                y = np.array([1 - 0.04 * t1, 0.04 * t1 * 1e-3]) + 1e-3 * rng.standard_normal(2)
            else:
                y = np.array([1.2])
            ys.append(y)
            anc, ll, g = R.ancestors(sc, ens, y, j, t0, t1)
            tr = R.pf_step(sc, ens, y, j, t0, t1)
            d[f"s{j}_anc"], d[f"s{j}_llbar"], d[f"s{j}_g"], d[f"s{j}_trace"] = anc, ll, g, tr
            for f in ("states", "params_u", "logw", "mean_u", "cov_u"):
                d[f"s{j}_{f}"] = getattr(ens, f).copy()
        d["ys"] = np.array(ys)
        np.savez_compressed(os.path.join(HERE, f"pf_{name}.npz"), **d)
        O.set_model_consts()
        R.set_model_consts()
        print("wrote", name)


def resample_cases():
    R = Reference()
    rng = np.random.default_rng(7)
    out = {}
    for name, g in [("uniform_1000", np.full(1000, 1e-3)),
                    ("lognormal_s1_5000", np.exp(rng.standard_normal(5000))),
                    ("lognormal_s4_5000", np.exp(4 * rng.standard_normal(5000))),
                    ("onehot_64", np.eye(64)[17])]:
        g = g / g.sum() if name != "onehot_64" else g
        out[name] = (g, R.resample(g, 99, 4))
    np.savez_compressed(os.path.join(HERE, "resample.npz"),
                        **{f"{k}_g": v[0] for k, v in out.items()}, **{f"{k}_anc": v[1] for k, v in out.items()})


if __name__ == "__main__":
    only = sys.argv[1:]  # optional case-name filter (pf cases only)
    if only:
        CASES = {k: v for k, v in CASES.items() if any(o in k for o in only)}
        pf_cases()
    else:
        philox_kats()
        streams()
        pf_cases()
        resample_cases()
