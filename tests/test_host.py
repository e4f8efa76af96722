"""Host-side checks that need no GPU: the C-ABI library loads and exports every
symbol include/pfsmc_gpu.h declares, the host Philox used for observation
noise equals the reference streams, problem generators are deterministic,
and the product refuses to run without a GPU (no CPU fallback)."""
import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
HEADERS = [os.path.join(ROOT, "include", h) for h in ("pfsmc_gpu.h", "pfsmc_gpu_experiment.h")]


def declared_symbols():
    txt = "".join(open(h).read() for h in HEADERS)
    return sorted(set(re.findall(r"\b(pfsmc_gpu_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    import ctypes
    from paper_1411_1702_b200.sampler import LIB_PATH
    lib = ctypes.CDLL(LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    lib.pfsmc_gpu_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.pfsmc_gpu_version()


def test_library_is_sm100a_only():
    import subprocess
    from paper_1411_1702_b200.sampler import LIB_PATH
    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_host_philox_matches_reference_streams():
    from paper_1411_1702_b200.problems import HostStream, philox4x64
    kats = json.load(open(os.path.join(GOLD, "philox_vectors.json")))["vectors"]
    for k in kats:
        out = philox4x64([int(x, 16) for x in k["ctr"]], [int(x, 16) for x in k["key"]])
        assert [f"{x:016x}" for x in out] == k["out"]
    st = json.load(open(os.path.join(GOLD, "rng_streams.json")))["streams"]
    for key, v in st.items():
        seed, j, n, purpose = map(int, key.split("_"))
        s = HostStream(seed, j, n, purpose)
        assert [f"{s.next_u64():016x}" for _ in range(9)] == v["u64"]
        s = HostStream(seed, j, n, purpose)
        assert [float.hex(s.next_normal()) for _ in range(9)] == v["normal"]


def test_problem_generators_are_deterministic():
    from paper_1411_1702_b200 import problems
    a = problems.lotka_volterra(particles=16, T=20, seed=3)
    b = problems.lotka_volterra(particles=16, T=20, seed=3)
    assert np.array_equal(a.ys, b.ys) and a.ys.shape == (20, 2)
    assert not np.array_equal(a.ys, problems.lotka_volterra(particles=16, T=20, seed=4).ys)
    r = problems.robertson(particles=16, T=50, seed=1)
    assert r.ys.shape == (50, 2) and np.all(r.ys > 0)
    c = problems.chain8(particles=16, T=30, seed=1)
    assert c.ys.shape == (30, 3)


def test_no_cpu_fallback_without_gpu():
    """The product path fails loudly when no device is visible."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    from paper_1411_1702_b200.sampler import GpuSampler, ObservationModel, PfConfig, PfsmcError
    with pytest.raises(PfsmcError):
        GpuSampler("lv", PfConfig(particles=16), ObservationModel([0, 1], 0.05))


def test_product_never_imports_oracle():
    """Only tests/, __graft_entry__.smoke and bench.py may touch oracle/."""
    pkg = os.path.join(ROOT, "paper_1411_1702_b200")
    bad = re.compile(r"oracle_ctypes|liboracle|libpfsmc_ref|oracle/|import oracle|from oracle")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                assert not bad.search(open(os.path.join(dp, f)).read()), f
