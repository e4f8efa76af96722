"""The experiment-level drop-in on the GPU against the unmodified reference's
pfsmc_run_experiment (oracle/_ref): same config, same data file (written by
the reference's pfsmc_generate_data), then the trace CSV row by row and the
report's fields. Free-running over the whole run: posterior mean / variance
rows within 1e-8, ESS within 1e-8."""
import ctypes as C
import csv
import json
import os

import numpy as np
import pytest

from oracle_ctypes import REF_SO

pytestmark = pytest.mark.gpu


def _libs():
    from paper_1411_1702_b200.sampler import LIB_PATH
    G = C.CDLL(LIB_PATH)
    G.pfsmc_gpu_experiment_new.restype = C.c_void_p
    G.pfsmc_gpu_experiment_last_error.restype = C.c_char_p
    R = C.CDLL(REF_SO)
    R.pfsmc_config_new.restype = C.c_void_p
    R.pfsmc_last_error.restype = C.c_char_p
    return G, R


def _rows(path):
    with open(path) as f:
        rd = list(csv.reader(f))
    return rd[0], np.array([[float(x) for x in r] for r in rd[1:]])


@pytest.mark.parametrize("kv", [
    [("particles", "2000"), ("integrator", "bdf2"), ("step", "0.05"), ("n-obs", "25"), ("t-end", "5"),
     ("seed", "11")],
    [("particles", "1500"), ("integrator", "am2"), ("step", "0.025"), ("n-obs", "12"), ("t-end", "3"),
     ("seed", "4"), ("const.tau", "0.8"), ("prior.k2.sigma", "0.3"), ("warmup", "1")],
    [("particles", "1000"), ("integrator", "adaptive-bdf2"), ("rtol", "1e-4"), ("n-obs", "15"), ("t-end", "3"),
     ("seed", "8")],
])
def test_run_experiment_matches_reference(kv, tmp_path, atol=0.0):
    G, R = _libs()
    g, r = C.c_void_p(G.pfsmc_gpu_experiment_new()), C.c_void_p(R.pfsmc_config_new())
    for k, v in kv:
        assert R.pfsmc_config_set(r, k.encode(), v.encode()) == 0
        assert G.pfsmc_gpu_experiment_set(g, k.encode(), v.encode()) == 0
    data = str(tmp_path / "data.csv")
    assert R.pfsmc_generate_data(r, data.encode()) == 0, R.pfsmc_last_error()
    ro, go = C.c_char_p(), C.c_char_p()
    assert R.pfsmc_run_experiment(r, data.encode(), str(tmp_path / "ref").encode(), C.byref(ro)) == 0
    rc = G.pfsmc_gpu_run_experiment(g, data.encode(), str(tmp_path / "gpu").encode(), C.byref(go))
    assert rc == 0, G.pfsmc_gpu_experiment_last_error()
    rep_r, rep_g = json.load(open(ro.value.decode())), json.load(open(go.value.decode()))
    assert rep_g["config"] == rep_r["config"] and rep_g["config_hash"] == rep_r["config_hash"]
    assert rep_g["truth"] == rep_r["truth"] and rep_g["param_names"] == rep_r["param_names"]
    assert rep_g["backend"] == "gpu" and os.path.basename(rep_g["trace_csv"]).endswith("_gpu.csv")
    hr, tr = _rows(rep_r["trace_csv"])
    hg, tg = _rows(rep_g["trace_csv"])
    assert hr == hg and tr.shape == tg.shape
    assert np.array_equal(tr[:, :2], tg[:, :2])  # j, t: identical text values
    np.testing.assert_allclose(tg[:, 2:], tr[:, 2:], rtol=1e-8, atol=atol)
    np.testing.assert_allclose(rep_g["final_estimate"], rep_r["final_estimate"], rtol=1e-8)
    np.testing.assert_allclose(rep_g["final_std_u"], rep_r["final_std_u"], rtol=1e-8, atol=np.sqrt(atol))
    assert rep_g["warnings"] == rep_r["warnings"]
    # PhaseTimings from the device (CUDA events per kernel)
    ph = rep_g["phases"]
    assert ph["propagate"] > 0 and ph["resample"] > 0 and ph["repropagate"] > 0, ph


def test_run_experiment_errors_match_reference(tmp_path):
    """Data-file and grid errors: same status codes as the reference."""
    G, R = _libs()
    g, r = C.c_void_p(G.pfsmc_gpu_experiment_new()), C.c_void_p(R.pfsmc_config_new())
    for lib, h, setter in ((G, g, G.pfsmc_gpu_experiment_set), (R, r, R.pfsmc_config_set)):
        setter(h, b"n-obs", b"6")
        setter(h, b"particles", b"100")
    data = str(tmp_path / "d.csv")
    assert R.pfsmc_generate_data(r, data.encode()) == 0
    for k, v in [("step", "0.07")]:  # does not divide the spacing
        G.pfsmc_gpu_experiment_set(g, k.encode(), v.encode())
        R.pfsmc_config_set(r, k.encode(), v.encode())
        o = C.c_char_p()
        a = G.pfsmc_gpu_run_experiment(g, data.encode(), str(tmp_path / "g").encode(), C.byref(o))
        b = R.pfsmc_run_experiment(r, data.encode(), str(tmp_path / "r").encode(), C.byref(o))
        assert a == b == 2
    # ragged data file
    with open(data, "a") as f:
        f.write("9.0,1.0\n")
    o = C.c_char_p()
    assert G.pfsmc_gpu_run_experiment(g, data.encode(), str(tmp_path / "g").encode(), C.byref(o)) == 4


@pytest.mark.parametrize("kv", [[("n-obs", "30"), ("t-end", "6"), ("seed", "21")],
                                [("n-obs", "10"), ("t-end", "4"), ("seed", "2"), ("const.A", "3.5"),
                                 ("truth.V1", "1.7"), ("x0.0.truth", "0.6"), ("sigma", "0.05")]])
def test_generate_data_matches_reference(kv, tmp_path):
    """pfsmc_gpu_generate_data vs the reference's pfsmc_generate_data: the truth
    path is integrated on the GPU (adaptive BDF(1,2), rtol 1e-8) and the noise
    comes from the same keyed streams, so every value agrees to rounding."""
    G, R = _libs()
    g, r = C.c_void_p(G.pfsmc_gpu_experiment_new()), C.c_void_p(R.pfsmc_config_new())
    for k, v in kv:
        assert R.pfsmc_config_set(r, k.encode(), v.encode()) == 0
        assert G.pfsmc_gpu_experiment_set(g, k.encode(), v.encode()) == 0
    dr, dg = str(tmp_path / "ref.csv"), str(tmp_path / "gpu.csv")
    assert R.pfsmc_generate_data(r, dr.encode()) == 0
    assert G.pfsmc_gpu_generate_data(g, dg.encode()) == 0, G.pfsmc_gpu_experiment_last_error()
    hr, vr = _rows(dr)
    hg, vg = _rows(dg)
    assert hr == hg and vr.shape == vg.shape
    assert np.array_equal(vr[:, 0], vg[:, 0])
    np.testing.assert_allclose(vg[:, 1:], vr[:, 1:], rtol=1e-10, atol=1e-12)
    sr, sg = json.load(open(dr[:-4] + ".json")), json.load(open(dg[:-4] + ".json"))
    assert set(sr) == set(sg)
    for key in sr:
        if key == "sigma":
            assert abs(sg[key] - sr[key]) <= 1e-10 * sr[key]
        else:
            assert sg[key] == sr[key], key
    # the GPU-generated file drives the reference's own experiment (format compatibility)
    o = C.c_char_p()
    assert R.pfsmc_run_experiment(r, dg.encode(), str(tmp_path / "o").encode(), C.byref(o)) == 0, \
        R.pfsmc_last_error()


# ---- the reference's problem 2 (AdvDiffModel), bench.cpp:249-277 ----------
@pytest.mark.parametrize("kv", [
    [("problem", "advdiff"), ("n", "6"), ("particles", "300"), ("integrator", "bdf2"), ("step", "0.05"),
     ("seed", "3")],
    [("problem", "advdiff"), ("n", "6"), ("particles", "48"), ("integrator", "adaptive-bdf2"), ("rtol", "1e-3"),
     ("seed", "1"), ("prior.k3.sigma", "1.5")],
])
def test_run_experiment_advdiff_matches_reference(kv, tmp_path):
    """Same data file (the reference's generator), free-running 30
    observations: trace rows within 1e-8, same report fields. The problem's
    tight noise (sigma = max|x0| / 50) collapses the posterior within a few
    observations; the collapsed variances are rounding noise (~1e-29), so
    they are compared with an absolute floor of 1e-12."""
    test_run_experiment_matches_reference(kv, tmp_path, atol=1e-12)


@pytest.mark.parametrize("kv", [[("problem", "advdiff"), ("n", "6"), ("seed", "5")],
                                [("problem", "advdiff"), ("n", "10"), ("seed", "1"), ("truth.c1", "1.5")]])
def test_generate_data_advdiff_matches_reference(kv, tmp_path):
    """pfsmc_gpu_generate_data for problem 2: the 20 random sites from the
    keyed stream and the noise are identical; the truth path is the adaptive
    BDF(1,2) at rtol 1e-8 on both sides (GPU: DFT Newton solve; reference: LU),
    so the values agree to the integrator's tolerance, not to rounding."""
    G, R = _libs()
    g, r = C.c_void_p(G.pfsmc_gpu_experiment_new()), C.c_void_p(R.pfsmc_config_new())
    for k, v in kv:
        assert R.pfsmc_config_set(r, k.encode(), v.encode()) == 0
        assert G.pfsmc_gpu_experiment_set(g, k.encode(), v.encode()) == 0
    dr, dg = str(tmp_path / "ref.csv"), str(tmp_path / "gpu.csv")
    assert R.pfsmc_generate_data(r, dr.encode()) == 0
    assert G.pfsmc_gpu_generate_data(g, dg.encode()) == 0, G.pfsmc_gpu_experiment_last_error()
    hr, vr = _rows(dr)
    hg, vg = _rows(dg)
    assert hr == hg and vr.shape == vg.shape == (30, 21)
    assert np.array_equal(vr[:, 0], vg[:, 0])
    np.testing.assert_allclose(vg[:, 1:], vr[:, 1:], rtol=0, atol=1e-7 * np.max(np.abs(vr[:, 1:])))
    sr, sg = json.load(open(dr[:-4] + ".json")), json.load(open(dg[:-4] + ".json"))
    assert set(sr) == set(sg)
    for key in sr:
        assert sg[key] == sr[key], key
