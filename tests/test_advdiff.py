"""The reference's problem 2, AdvDiffModel (models.cpp:158-266), on the CPU
checkers: the C oracle's restatement (CSR operator assembly, spmv, the
sparse Newton path with its per-workspace factorisation) is bitwise equal to
the unmodified reference (oracle/_ref, Eigen's SparseLU replaced by the
stand-in direct LU of oracle/ref/eigen_stub), and the 7-point stencil the GPU
kernels use (csrc/advdiff.cuh adv_stencil) reproduces the reference's CSR
values bit for bit. The GPU side is tests/test_advdiff_gpu.py.
"""
import ctypes as C
import os

import numpy as np
import pytest

from oracle_ctypes import (METABOLIC_DEFAULTS, REF_SO, Oracle, Reference, StepConfig,
                           set_advdiff_grid)

O = Oracle()
TRUTH = np.array([9.0, 4.0, 6.0, 2.5, -1.5])  # bench.cpp:251-255
needs_ref = pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")


@pytest.fixture(autouse=True)
def _reset_consts():
    yield
    O.set_model_consts(METABOLIC_DEFAULTS)


def plume(n):
    x0 = np.zeros((n - 1) ** 2)
    O.lib.or_gaussian_plume_ic(n, x0.ctypes.data_as(C.POINTER(C.c_double)))
    return x0


def dense_operator(n, th):
    d = (n - 1) ** 2
    out = np.zeros((d, d))
    th = np.ascontiguousarray(th, dtype=np.float64)
    assert O.lib.or_advdiff_operator(n, th.ctypes.data_as(C.POINTER(C.c_double)),
                                     out.ctypes.data_as(C.POINTER(C.c_double))) == 0
    return out


def stencil(th):
    """adv_stencil (csrc/advdiff.cuh) in Python: csr_add's value rule over
    the Gram / difference stencils (linalg.cpp:142-180, models.cpp:251-261)."""
    k1, k2, k3, c1, c2 = th
    A, B, Cc = -(k1 * k1), -(k1 * k3), -(k2 * k2 + k3 * k3)
    g11 = {(0, 0): 2.0, (-1, 0): -1.0, (1, 0): -1.0}
    g22 = {(0, 0): 2.0, (0, -1): -1.0, (0, 1): -1.0}
    g12 = {(0, 0): 2.0, (0, -1): -1.0, (1, 0): -1.0, (1, -1): 1.0, (-1, 0): -1.0, (0, 1): -1.0, (-1, 1): 1.0}
    b1 = {(0, 0): 1.0, (-1, 0): -1.0}
    b2 = {(0, 0): 1.0, (0, -1): -1.0}

    def add(al, a, be, b):
        out = {}
        for o in set(a) | set(b):
            if o in a:
                v = 0.0 + al * a[o]
                if o in b:
                    v = v + be * b[o]
            else:
                v = be * b[o]
            out[o] = v
        return out

    return add(1.0, add(1.0, add(A, g11, B, g12), Cc, g22), 1.0, add(c1, b1, c2, b2))


@pytest.mark.parametrize("n", [4, 5, 8, 20])
def test_stencil_matches_reference_operator_bitwise(n):
    m = n - 1
    rng = np.random.default_rng(n)
    for th in (TRUTH, rng.normal(size=5) * 5):
        L = dense_operator(n, th)
        D = np.zeros_like(L)
        for (dx, dy), v in stencil(th).items():
            for iy in range(m):
                for ix in range(m):
                    D[iy * m + ix, ((iy + dy) % m) * m + (ix + dx) % m] += v
        assert np.array_equal(L, D)


def test_operator_structure():
    """acceptance_main.cpp:376-410 (criterion C5): the operator annihilates
    constants and its columns sum to zero (mass conservation)."""
    for n in (5, 20):
        L = dense_operator(n, TRUTH)
        assert np.max(np.abs(L @ np.ones(L.shape[0]))) < 1e-10
        assert np.max(np.abs(L.sum(axis=0))) < 1e-10


def test_spectrum_diagonalises_operator():
    """The GPU solve's premise: L is block-circulant with circulant blocks,
    so the 2-D DFT diagonalises it with eigenvalues sum_o s_o e^{2 pi i k.o/m}."""
    n = 7
    m = n - 1
    L = dense_operator(n, TRUTH)
    s = stencil(TRUTH)
    lam = np.zeros((m, m), complex)
    for (dx, dy), v in s.items():
        for ky in range(m):
            for kx in range(m):
                lam[ky, kx] += v * np.exp(2j * np.pi * (kx * dx + ky * dy) / m)
    hb0 = 0.05 * 2.0 / 3.0
    r = np.random.default_rng(1).normal(size=m * m)
    x_dft = np.real(np.fft.ifft2(np.fft.fft2(r.reshape(m, m)) / (1 - hb0 * lam))).ravel()
    x_lu = np.linalg.solve(np.eye(m * m) - hb0 * L, r)
    assert np.max(np.abs(x_dft - x_lu)) < 1e-13 * np.max(np.abs(x_lu))


@needs_ref
@pytest.mark.parametrize("n", [4, 6, 10])
@pytest.mark.parametrize("family,order", [("ab", 2), ("am", 1), ("am", 3), ("bdf", 1), ("bdf", 2), ("bdf", 3)])
def test_oracle_propagate_matches_reference_bitwise(n, family, order):
    R = Reference()
    set_advdiff_grid(n, O, R)
    try:
        x0 = plume(n)
        h = 0.001 if family == "ab" else 0.05
        a = O.propagate("advdiff", TRUTH, x0, 0.0, 1.0, h, family, order)
        b = R.propagate("advdiff", TRUTH, x0, 0.0, 1.0, h, family, order)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        assert a[2:] == b[2:]
    finally:
        R.set_model_consts(METABOLIC_DEFAULTS)


@needs_ref
@pytest.mark.parametrize("n,family,order,adaptive", [(6, "bdf", 2, False), (5, "am", 3, False),
                                                     (7, "bdf", 3, False), (6, "bdf", 2, True)])
def test_oracle_pf_step_matches_reference_bitwise(n, family, order, adaptive):
    R = Reference()
    set_advdiff_grid(n, O, R)
    try:
        d = (n - 1) ** 2
        x0 = plume(n)
        idx = tuple(int(v) % d for v in (3, 7, 11, 20, 24))
        sc = StepConfig(model="advdiff", family=family, order=order, h=0.05, a=0.98, seed=5, obs_idx=idx,
                        sigma=float(x0.max() / 10), adaptive=adaptive)
        ens = R.init_gaussian(sc, 64, [np.log(7), np.log(5), 4, 0, 0], [0.35, 0.35, 2, 2, 2], x0,
                              np.zeros(d), np.zeros(d, np.int32))
        eo = O.init_gaussian("advdiff", 64, 5, [np.log(7), np.log(5), 4, 0, 0], [0.35, 0.35, 2, 2, 2], x0,
                             np.zeros(d), np.zeros(d, np.int32))
        for f in ("states", "params_u", "logw", "mean_u", "cov_u"):
            assert np.array_equal(getattr(ens, f), getattr(eo, f)), f
        rng = np.random.default_rng(0)
        xt = x0.copy()
        for j in range(1, 4):
            xt = O.propagate("advdiff", TRUTH, xt, j - 1.0, float(j), 0.01, "bdf", 2)[0]
            y = xt[list(idx)] + sc.sigma * rng.standard_normal(len(idx))
            tr = R.pf_step(sc, ens, y, j, j - 1.0, float(j))
            to, _ = O.pf_step(sc, eo, y, j, j - 1.0, float(j))
            assert np.array_equal(tr, to)
            for f in ("states", "params_u", "logw", "mean_u", "cov_u"):
                assert np.array_equal(getattr(ens, f), getattr(eo, f)), (j, f)
    finally:
        R.set_model_consts(METABOLIC_DEFAULTS)
