"""Pins for oracle.eigsolve (inverse Lanczos + CG)
against the plain definition (dense GEP / dense NFSEP eigh)."""
import json
import os

import numpy as np
import pytest

from oracle import eigsolve, fftop, lattice, spectral
from synthetic import configs
from synthetic import eps as E


def test_cg_solves_hpd_system():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((40, 40)) + 1j * rng.standard_normal((40, 40))
    A = A.conj().T @ A + 40 * np.eye(40)
    b = rng.standard_normal(40) + 0j
    x, its = eigsolve.cg(lambda v: A @ v, b, tol=1e-13)
    assert np.linalg.norm(A @ x - b) <= 1.01e-13 * np.linalg.norm(b)


def test_config1_inverse_lanczos_matches_dense_gep(golden_dir):
    """Config 1 (SC 12^3 sphere): the paper's solver reproduces the 10
    smallest nonzero GEP eigenvalues of the dense plain definition
    (tests/golden/config1_dense_oracle.json) to 1e-10 relative."""
    with open(os.path.join(golden_dir, "config1_dense_oracle.json")) as f:
        gold = json.load(f)
    cfg = configs.config(1)
    L = lattice.snap(cfg.a_raw, cfg.n)
    eps = E.sample(cfg.shape, cfg.n, L.a, L.delta, L.a_canon)
    kap = lattice.kvec_reduce(L, cfg.kpoints[0])
    op = fftop.NFSEPOperator(L, kap, eps)
    lam, Y, info = eigsolve.inverse_lanczos(op, nev=10, block=2, guard=2)
    np.testing.assert_allclose(lam, gold["lambda"][:10], rtol=1e-10)
    for i in range(10):
        r = op.Ar(Y[:, i]) - lam[i] * Y[:, i]
        assert np.linalg.norm(r) / np.linalg.norm(Y[:, i]) < 1e-6


def test_block_lanczos_finds_degenerate_copy():
    """at the simple-cubic X point eigenvalues are exactly
    degenerate; a block Krylov basis (b=4) finds every copy the dense
    NFSEP eigh finds."""
    L = lattice.snap(configs.sc_vectors(), (6, 6, 6))
    eps = E.sample("sc_sphere", L.n, L.a, L.delta, L.a_canon)
    kap = (0.5, 0.0, 0.0)
    dense = np.linalg.eigvalsh(spectral.Ar_dense(L, kap, eps))[:8]
    op = fftop.NFSEPOperator(L, kap, eps)
    lam, _, _ = eigsolve.inverse_lanczos(op, nev=8, block=4, guard=4)
    np.testing.assert_allclose(lam, dense, rtol=1e-10)
    assert np.sum(np.abs(np.diff(dense)) < 1e-9 * dense[-1]) >= 2    # degeneracies present


@pytest.mark.parametrize("case", range(9))
def test_small_config_lattices(golden_dir, case):
    """Oracle solver vs dense NFSEP on the config lattices at small grids
    (tests/golden/small_nfsep_oracle.json), including Gamma (masked)."""
    with open(os.path.join(golden_dir, "small_nfsep_oracle.json")) as f:
        c = json.load(f)["cases"][case]
    cfg = configs.config(c["config"])
    n = tuple(c["n"])
    L = lattice.snap(cfg.a_raw, n)
    eps = E.sample(cfg.shape, n, L.a, L.delta, L.a_canon)
    op = fftop.NFSEPOperator(L, tuple(c["kappa"]), eps)
    nev = 6
    lam, _, _ = eigsolve.inverse_lanczos(op, nev=nev, block=4, guard=4)
    np.testing.assert_allclose(lam, c["lambda"][:nev], rtol=1e-10)


@pytest.mark.parametrize("case", [0, 4, 8])
def test_arpack_route_matches_dense(golden_dir, case):
    """The bounded-memory ARPACK route (used for the 256^3 golden) reaches
    the dense NFSEP eigenvalues (tests/golden/small_nfsep_oracle.json) to
    1e-10 relative, including a masked Gamma case."""
    with open(os.path.join(golden_dir, "small_nfsep_oracle.json")) as f:
        c = json.load(f)["cases"][case]
    cfg = configs.config(c["config"])
    n = tuple(c["n"])
    L = lattice.snap(cfg.a_raw, n)
    eps = E.sample(cfg.shape, n, L.a, L.delta, L.a_canon)
    op = fftop.NFSEPOperator(L, tuple(c["kappa"]), eps)
    lam, Y, _ = eigsolve.arpack_inverse(op, nev=6, guard=4)
    np.testing.assert_allclose(lam, c["lambda"][:6], rtol=1e-10)
    for i in range(6):
        r = op.Ar(Y[:, i]) - lam[i] * Y[:, i]
        assert np.linalg.norm(r) / np.linalg.norm(Y[:, i]) < 1e-6


def test_threaded_operator_bit_identical():
    """ORACLE_THREADS / ORACLE_FFT_WORKERS change only execution: the
    threaded M equals the serial M bit for bit."""
    from oracle import fftop as F
    cfg = configs.config(4)
    n = (12, 10, 8)
    L = lattice.snap(cfg.a_raw, n)
    eps = E.sample(cfg.shape, n, L.a, L.delta, L.a_canon)
    op = F.NFSEPOperator(L, (0.1, 0.2, 0.3), eps)
    y = np.random.default_rng(1).standard_normal(2 * op.n) + 1j
    z0 = op.M(y)
    t, w = F._THREADS, F._WORKERS
    try:
        F._THREADS, F._WORKERS = 3, 2
        z1 = op.M(y)
    finally:
        F._THREADS, F._WORKERS = t, w
    assert np.array_equal(z0, z1)


@pytest.mark.parametrize("which", ["sc", "fcc", "bcc_gamma", "triclinic"])
def test_recover_satisfies_sparse_gep(which):
    """oracle.fftop.NFSEPOperator.recover: for an eigenpair
    A_r y = lambda y (dense NFSEP eigh), e = B^{-1} Q_r Sigma_r y solves the
    GEP of the independently assembled sparse Yee curl (oracle.curl,
    geometric wrap): C^*C e = lambda B e, with e^* B e = lambda y^* y.
    (C^*C = Q_r Sigma_r^2 Q_r^* by the SVD theorem.)"""
    cases = {"sc": (configs.sc_vectors(), (5, 4, 6), "random:1", (0.21, -0.13, 0.4)),
             "fcc": (configs.fcc_vectors(), (6, 6, 5), "fcc_diamond", (0.5, 0.25, 0.75)),
             "bcc_gamma": (configs.bcc_vectors(), (6, 6, 4), "bcc_sphere_rod", (0.0, 0.0, 0.0)),
             "triclinic": (configs.triclinic_vectors(), (6, 5, 7), "random:5", (0.2, -0.3, 0.45))}
    a, n, shape, kap = cases[which]
    from oracle import curl
    L = lattice.snap(a, n)
    eps = E.sample(shape, n, L.a, L.delta, L.a_canon)
    op = fftop.NFSEPOperator(L, kap, eps)
    w, Y = np.linalg.eigh(spectral.Ar_dense(L, kap, eps))
    C = curl.curl(L, kap)
    Bd = curl.B_diag(eps)
    first = 2 if which == "bcc_gamma" else 0          # masked Gamma mode: 2 structural zeros (R6)
    for i in range(first, first + 5):
        lam, y = w[i], Y[:, i]
        e = op.recover(y).ravel()
        res = np.linalg.norm(C.conj().T @ (C @ e) - lam * Bd * e) / (lam * np.linalg.norm(Bd * e))
        assert res < 1e-11, (which, i, res)
        np.testing.assert_allclose(np.vdot(e, Bd * e).real, lam * np.vdot(y, y).real, rtol=1e-11)
