"""Pins for oracle.curl (§3): the geometric-wrap curl against the
paper's explicit block forms, structural identities, the null-space
dimension and the dense GEP definition."""
import math

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import curl, lattice
from synthetic import configs


def random_lattices(count, seed=7, nmax=7):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        try:
            a = configs.triclinic_vectors(1.0, rng.uniform(0.6, 1), rng.uniform(0.6, 1),
                                          *rng.uniform(50, 130, 3))
            L = lattice.snap(a, tuple(int(x) for x in rng.integers(3, nmax + 1, 3)))
        except ValueError:
            continue
        out.append((L, tuple(rng.uniform(-0.5, 0.5, 3))))
    return out


def _psi_boundary(L):
    n1 = L.n[0]
    m1, m2, _ = L.m
    r1, r2, r3 = L.rho
    s1 = (r2 * n1 - m2) - (r1 * n1 - m1)
    s2 = (r1 * n1 - m1) + (r2 * n1 - m2)
    return (r3 == 0 and s1 == 0) or (r3 == 1 and s2 == 0)


def test_K1_K2_match_paper_forms():
    """C1 = I (x) I (x) K1, C2 = I (x) K2 with general J2."""
    for L, kap in random_lattices(60):
        n1, n2, n3 = L.n
        C1, C2, _ = curl.partials(L, kap)
        np.testing.assert_allclose(C1.toarray(), np.kron(np.eye(n2 * n3), curl.K1_paper(L, kap)), atol=1e-12)
        np.testing.assert_allclose(C2.toarray(), np.kron(np.eye(n3), curl.K2_paper(L, kap)), atol=1e-12)


def test_K3_matches_paper_four_categories():
    """C3 = K3 with the four general J3 categories, away from the
    psi-flag boundary ((rho2 n1 - m2) - (rho1 n1 - m1) = 0 resp.
    (rho1 n1 - m1) + (rho2 n1 - m2) = 0) where the printed flags are
    ambiguous (R14)."""
    seen = set()
    checked = 0
    for L, kap in random_lattices(400, seed=11):
        if _psi_boundary(L):
            continue
        C3 = curl.partials(L, kap)[2].toarray()
        np.testing.assert_allclose(C3, curl.K3_paper(L, kap), atol=1e-9 / L.delta[2] * 1e-3)
        seen.add(curl.J3_category(L))
        checked += 1
    assert seen == {1, 2, 3, 4} and checked > 100


def test_sc_kappa0_is_periodic_difference():
    """SC, kappa = 0: C1 is the periodic forward difference (textbook)."""
    L = lattice.snap(configs.sc_vectors(), (5, 4, 3))
    C1 = curl.partials(L, (0.0, 0.0, 0.0))[0].toarray() * L.delta[0]
    D = -np.eye(5) + np.roll(np.eye(5), 1, axis=1)
    np.testing.assert_allclose(C1, np.kron(np.eye(12), D), atol=0)


def test_commuting_partials_and_curl_structure():
    """C_i C_j = C_j C_i ('commute to each other'); C^* C Q0 = 0
    follows; div(curl) = 0 on the E side: [C1 C2 C3] C = 0 (H-side) ."""
    for L, kap in random_lattices(12, seed=3):
        C = curl.partials(L, kap)
        for i in range(3):
            for j in range(i + 1, 3):
                d = (C[i] @ C[j] - C[j] @ C[i])
                assert abs(d).max() <= 1e-9 * max(1.0, abs(C[i]).max() * abs(C[j]).max()) * 1e-3
        CC = curl.curl(L, kap)
        G = sp.hstack(C)
        assert abs(G @ CC).max() <= 1e-12 * abs(CC).max() ** 2


@pytest.mark.parametrize("kap,extra", [((0.21, -0.33, 0.4), 0), ((0.0, 0.0, 0.0), 2)])
def test_null_space_dimension(kap, extra):
    """dim null(C^*C) = n, n + 2 at Gamma (R6)."""
    for L, _ in random_lattices(4, seed=5, nmax=5):
        eps = [1.0 + np.random.default_rng(1).random(L.nn) for _ in range(3)]
        _, nz, nnull = curl.dense_gep(L, kap, eps)
        assert nnull == L.nn + extra
        assert len(nz) == 2 * L.nn - extra


def test_dense_gep_vacuum_closed_form():
    """eps == c: nonzero GEP eigenvalues are 4 sum_l sin^2(pi g_l)/delta_l^2 / c
    (discrete free photon), each twice; SC kappa=(.25,.15,.05) plane waves."""
    L = lattice.snap(configs.sc_vectors(), (4, 3, 5))
    kap = (0.25, 0.15, 0.05)
    c = 2.5
    _, nz, _ = curl.dense_gep(L, kap, [np.full(L.nn, c)] * 3)
    i, j, k = np.meshgrid(np.arange(4), np.arange(3), np.arange(5), indexing="ij")
    g = [(i + kap[0]) / 4, (j + kap[1]) / 3, (k + kap[2]) / 5]
    q = sum(4 * np.sin(math.pi * gl) ** 2 / d ** 2 for gl, d in zip(g, L.delta)).ravel()
    np.testing.assert_allclose(np.sort(nz), np.sort(np.concatenate([q, q])) / c, rtol=1e-10)
