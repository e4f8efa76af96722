"""The experiment-level drop-in (include/pfsmc_gpu_experiment.h) on the host:
config keys, validation messages / status codes and the canonical config
JSON + FNV-1a hash, against the unmodified reference's experiment ABI
(pfsmc_config_set / pfsmc_run_experiment in oracle/_ref). No GPU needed."""
import ctypes as C
import json
import os

import pytest

from oracle_ctypes import REF_SO

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HAVE_REF = os.path.exists(REF_SO)


def _gpu_lib():
    from paper_1411_1702_b200.sampler import LIB_PATH
    L = C.CDLL(LIB_PATH)
    L.pfsmc_gpu_experiment_new.restype = C.c_void_p
    L.pfsmc_gpu_experiment_last_error.restype = C.c_char_p
    return L


def _ref_lib():
    L = C.CDLL(REF_SO)
    L.pfsmc_config_new.restype = C.c_void_p
    L.pfsmc_last_error.restype = C.c_char_p
    return L


CONFIGS = [
    [],
    [("particles", "500"), ("integrator", "am3"), ("step", "0.025"), ("n-obs", "20"), ("t-end", "4"),
     ("seed", "3"), ("prior.V1.sigma", "0.4"), ("const.tau", "0.7"), ("x0.1.mean", "1.3"), ("warmup", "true")],
    [("shrink-a", "0.95"), ("sigma", "0.125"), ("rtol", "1e-05"), ("backend", "par"), ("workers", "8"),
     ("truth.V1", "2.5"), ("n", "7")],
    # number layouts of the JSON writer: fixed / 0.000d / scientific boundaries
    # (unused override names carry the extreme values into the canonical JSON only)
    [("rtol", "1e-4"), ("truth.Za", "0.0001234"), ("truth.Zb", "1e15"), ("truth.Zc", "123456789012345678"),
     ("truth.Zd", "-2.5e-300"), ("truth.Ze", "1e16"), ("truth.Zf", "-0.0"), ("integrator", "adaptive-bdf2")],
]


@pytest.mark.parametrize("kv", CONFIGS)
def test_canonical_config_and_hash_match_reference(kv, tmp_path):
    if not HAVE_REF:
        pytest.skip("oracle/_ref not built")
    G, R = _gpu_lib(), _ref_lib()
    g, r = C.c_void_p(G.pfsmc_gpu_experiment_new()), C.c_void_p(R.pfsmc_config_new())
    for k, v in kv:
        assert G.pfsmc_gpu_experiment_set(g, k.encode(), v.encode()) == 0
        assert R.pfsmc_config_set(r, k.encode(), v.encode()) == 0
    js, hs = C.c_char_p(), C.c_char_p()
    assert G.pfsmc_gpu_experiment_canonical(g, C.byref(js), C.byref(hs)) == 0
    mine, my_hash = js.value.decode(), hs.value.decode()
    # the reference's report carries its canonical config and hash
    R.pfsmc_config_set(r, b"n-obs", b"5")
    R.pfsmc_config_set(r, b"particles", b"64")
    data = str(tmp_path / "d.csv")
    assert R.pfsmc_generate_data(r, data.encode()) == 0, R.pfsmc_last_error()
    out = C.c_char_p()
    assert R.pfsmc_run_experiment(r, data.encode(), str(tmp_path / "o").encode(), C.byref(out)) == 0, \
        R.pfsmc_last_error()
    rep = json.load(open(out.value.decode()))
    ref_cfg = dict(rep["config"])
    want = json.loads(mine)
    want["n_obs"], want["particles"] = 5, 64  # the two keys changed for the quick reference run
    assert ref_cfg == want
    G.pfsmc_gpu_experiment_set(g, b"n-obs", b"5")
    G.pfsmc_gpu_experiment_set(g, b"particles", b"64")
    assert G.pfsmc_gpu_experiment_canonical(g, C.byref(js), C.byref(hs)) == 0
    assert hs.value.decode() == rep["config_hash"], (js.value, rep["config"])
    G.pfsmc_gpu_experiment_free(g)
    R.pfsmc_config_free(r)


def test_config_errors_match_reference():
    G = _gpu_lib()
    R = _ref_lib() if HAVE_REF else None
    g = C.c_void_p(G.pfsmc_gpu_experiment_new())
    r = C.c_void_p(R.pfsmc_config_new()) if R else None
    for k, v in [("problem", "other"), ("integrator", "ab4"), ("backend", "gpu"), ("particles", "12x"),
                 ("step", "abc"), ("nonsense", "1")]:
        rc = G.pfsmc_gpu_experiment_set(g, k.encode(), v.encode())
        assert rc == 2, (k, v)
        msg = G.pfsmc_gpu_experiment_last_error().decode()
        if R:
            assert R.pfsmc_config_set(r, k.encode(), v.encode()) == 2
            assert msg == R.pfsmc_last_error().decode()
    G.pfsmc_gpu_experiment_free(g)


def test_problem_validation_and_missing_data_status(tmp_path):
    G = _gpu_lib()
    g = C.c_void_p(G.pfsmc_gpu_experiment_new())
    out = C.c_char_p()
    # missing data file: IO error before any GPU work
    assert G.pfsmc_gpu_run_experiment(g, str(tmp_path / "none.csv").encode(), str(tmp_path).encode(),
                                      C.byref(out)) == 4
    # problem 2 (AdvDiffModel): the grid bound of the GPU path is a CONFIG error, like the
    # reference's AdvDiffModel ctor for n < 3 (models.cpp:186-188); the data file is read first
    assert G.pfsmc_gpu_experiment_set(g, b"problem", b"advdiff") == 0
    assert G.pfsmc_gpu_experiment_set(g, b"n", b"2") == 0
    assert G.pfsmc_gpu_run_experiment(g, str(tmp_path / "none.csv").encode(), str(tmp_path).encode(),
                                      C.byref(out)) == 2
    assert b"grid parameter n" in G.pfsmc_gpu_experiment_last_error()
    assert G.pfsmc_gpu_experiment_set(g, b"problem", b"other") == 2
    G.pfsmc_gpu_experiment_free(g)
