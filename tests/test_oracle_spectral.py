"""Pins for oracle.spectral / oracle.fftop (§4-5): theorem
residuals against the independently built curl, unitarity, the textbook
DFT special case, SVD identities, and the null-space-free theorem by brute
force."""
import math

import numpy as np
import pytest

from oracle import curl, fftop, lattice, spectral
from synthetic import configs
from synthetic import eps as E
from tests.test_oracle_curl import random_lattices


def test_K1_eigenvalues_worked_example():
    """S:L236 / Thm eigK1: n1=4, k.a1=0, dx=1 ->
    {0, i-1, -2, -i-1}."""
    a = np.diag([4.0, 3.0, 3.0])        # dx = 4/4 = 1
    L = lattice.snap(a, (4, 3, 3))
    l1 = spectral.lambdas(L, (0.0, 0.0, 0.0))[0][0, 0, :]
    np.testing.assert_allclose(l1, [0, 1j - 1, -2, -1j - 1], atol=1e-15)


def test_theorem_residuals_all_categories():
    """C_l T = T Lambda_l with T, Lambda from the closed forms
    of Thms eigK1/eigK2/eigK3 and C from the geometric wrap: the two
    constructions share nothing but the lattice integers."""
    cats = set()
    for L, kap in random_lattices(40, seed=21):
        C = curl.partials(L, kap)
        T = spectral.T_dense(L, kap)
        lam = [x.ravel() for x in spectral.lambdas(L, kap)]
        for l in range(3):
            r = np.abs(C[l] @ T - T * lam[l][None, :]).max() * L.delta[l]
            assert r < 1e-13
        np.testing.assert_allclose(T.conj().T @ T, np.eye(L.nn), atol=1e-13)
        cats.add((L.rho, curl.J3_category(L)))
    assert len(cats) >= 6


def test_swapped_branch_fails():
    """R1: using the obtuse coefficient on an acute lattice breaks the
    residual (the P:L2035/L2041 conditions are swapped)."""
    for L, kap in random_lattices(40, seed=23):
        if L.rho[2] == 0 and L.m[0] > 0:
            break
    C3 = curl.partials(L, kap)[2]
    L.rho = (L.rho[0], L.rho[1], 1)
    T = spectral.T_dense(L, kap)
    lam = spectral.lambdas(L, kap)[2].ravel()
    assert np.abs(C3 @ T - T * lam[None, :]).max() * L.delta[2] > 1e-3


def test_T_is_textbook_dft_for_sc_kappa0():
    """Orthogonal lattice, kappa = 0: T q = sqrt(n) * ifftn(q)."""
    L = lattice.snap(configs.sc_vectors(), (4, 6, 5))
    T = spectral.T_dense(L, (0.0, 0.0, 0.0))
    q = np.random.default_rng(0).standard_normal((5, 6, 4)) + 0j
    want = np.fft.ifftn(q) * math.sqrt(L.nn)
    np.testing.assert_allclose(T @ q.ravel(), want.ravel(), atol=1e-12)


def test_fft_algorithms_match_dense_T():
    """Algorithms 1-2 equal dense T^* / T (different code:
    numpy FFTs + diagonal phases vs closed-form matrix)."""
    for L, kap in random_lattices(10, seed=31):
        T = spectral.T_dense(L, kap)
        x = np.random.default_rng(1).standard_normal(L.nn) + 1j
        shp = (L.n[2], L.n[1], L.n[0])
        np.testing.assert_allclose(fftop.T_apply(L, kap, x.reshape(shp)).ravel(), T @ x, atol=1e-12)
        np.testing.assert_allclose(fftop.Tstar_apply(L, kap, x.reshape(shp)).ravel(), T.conj().T @ x, atol=1e-12)


def test_gram_and_svd():
    """[Pi1 Pi2 Pi0] orthonormal per mode (Q, P unitary);
    C = P_r Sigma_r Q_r^* (eq. SVD) and C^*C Q0 = 0."""
    for L, kap in random_lattices(8, seed=41, nmax=5):
        Pi0, Pi1, Pi2, q = spectral.pis(L, kap)
        G = np.stack([Pi1, Pi2, Pi0])
        gram = np.einsum("aln,bln->abn", G.conj(), G)
        np.testing.assert_allclose(gram, np.broadcast_to(np.eye(3)[:, :, None], gram.shape), atol=1e-13)
        C = curl.curl(L, kap).toarray()
        Q0, Q1, Q2 = spectral.Q_dense(L, kap)
        P0, P1, P2 = spectral.P_dense(L, kap)
        Qr = np.concatenate([Q1, Q2], axis=1)
        Pr = np.concatenate([P2, P1], axis=1)
        s = np.sqrt(np.concatenate([q, q]))
        np.testing.assert_allclose(C, (Pr * s[None, :]) @ Qr.conj().T, atol=1e-10 * np.abs(C).max())
        assert np.abs(C @ Q0).max() < 1e-12 * np.abs(C).max()


def _cases():
    return [
        ("sc generic", configs.sc_vectors(), (4, 4, 4), (0.25, 0.15, 0.05), "random:3"),
        ("sc [111] Pi fallback (R5)", configs.sc_vectors(), (4, 4, 4), (0.1, 0.1, 0.1), "random:4"),
        ("sc Gamma (R6)", configs.sc_vectors(), (4, 4, 4), (0.0, 0.0, 0.0), "random:5"),
        ("fcc X diamond", configs.fcc_vectors(), (6, 6, 6), (0.5, 0.0, 0.5), "fcc_diamond"),
        ("bcc Gamma spheres+rods", configs.bcc_vectors(), (6, 6, 4), (0.0, 0.0, 0.0), "bcc_sphere_rod"),
        ("bcc H", configs.bcc_vectors(), (6, 6, 4), (0.5, -0.5, 0.5), "random:6"),
        ("triclinic", configs.triclinic_vectors(), (5, 4, 6), (0.2, -0.3, 0.45), "random:7"),
    ]


@pytest.mark.parametrize("name,a,n,kap,shape", _cases())
def test_nfsep_spectrum_equals_gep(name, a, n, kap, shape):
    """Null-space-free theorem: eig(A_r) = nonzero eig of
    C^*C e = lambda B e, brute force; A_r Hermitian; the matrix-free
    Algorithms-1/2 operator equals the dense A_r."""
    L = lattice.snap(a, n)
    eps = E.sample(shape, n, L.a, L.delta, L.a_canon)
    _, nz, nnull = curl.dense_gep(L, kap, eps)
    Ar = spectral.Ar_dense(L, kap, eps)
    assert np.abs(Ar - Ar.conj().T).max() <= 1e-14 * np.abs(Ar).max()
    ev = np.linalg.eigvalsh(Ar)
    g = spectral.gamma_mode(L, kap)
    if g is not None:
        assert nnull == L.nn + 2
        assert np.all(np.abs(ev[:2]) < 1e-10 * ev[-1])
        ev = ev[2:]
    np.testing.assert_allclose(ev, np.sort(nz), rtol=1e-11, atol=1e-12 * ev[-1])
    op = fftop.NFSEPOperator(L, kap, eps)
    y = np.random.default_rng(2).standard_normal(2 * L.nn) + 0.5j
    np.testing.assert_allclose(op.Ar(y), Ar @ y, atol=1e-12 * np.abs(Ar @ y).max())
    M = spectral.Ar_dense(L, kap, eps, op="M")
    np.testing.assert_allclose(op.M(y), M @ y, atol=1e-12 * np.abs(M @ y).max())


def test_fallback_actually_triggers():
    L = lattice.snap(configs.sc_vectors(), (4, 4, 4))
    lam = np.stack([x.ravel() for x in spectral.lambdas(L, (0.1, 0.1, 0.1))])
    lp = np.stack([lam[2] - lam[1], lam[0] - lam[2], lam[1] - lam[0]])
    assert np.sum(np.sum(np.abs(lp) ** 2, 0) <= spectral.TAU_P * np.sum(np.abs(lam) ** 2, 0)) == 4


def test_vacuum_Ar_is_sigma_squared():
    """eps == c: A_r = Sigma_r^2 / c exactly."""
    L = lattice.snap(configs.fcc_vectors(), (5, 4, 6))
    kap = (0.3, 0.1, -0.2)
    c = 3.0
    Ar = spectral.Ar_dense(L, kap, E.sample("vacuum:3.0", L.n))
    _, _, _, q = spectral.pis(L, kap)
    np.testing.assert_allclose(Ar, np.diag(np.concatenate([q, q]) / c), atol=1e-12 * q.max())
    np.testing.assert_allclose(np.linalg.eigvalsh(Ar), spectral.free_photon(L, kap, c), rtol=1e-12, atol=1e-10)


def test_condition_bound():
    """kappa(Q_r^* B^{-1} Q_r) <= kappa(B^{-1})."""
    L = lattice.snap(configs.triclinic_vectors(), (4, 5, 4))
    eps = E.sample("random:9", L.n)
    M = spectral.Ar_dense(L, (0.1, 0.2, 0.3), eps, op="M")
    w = np.linalg.eigvalsh(M)
    e = np.concatenate([x.ravel() for x in eps])
    assert w[-1] / w[0] <= e.max() / e.min() * (1 + 1e-12)
    assert w[0] >= 1 / e.max() * (1 - 1e-12) and w[-1] <= 1 / e.min() * (1 + 1e-12)
