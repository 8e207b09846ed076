"""Yee discrete curl and the GEP: PAPER.md §3 (L296-1646).  Test
infrastructure only.

Vectors are stored x-fastest: index(a, b, c) = a + n1*(b + n2*c)
(= vec() of P:L331 with i fastest).

Primary construction (``shift``/``partials``): the forward differences
C_l = (S_l - I)/delta_l of P:L343-378, where the shift S_l moves one grid
step along axis l and a neighbour leaving the box is brought back by the
quasi-periodic condition E(x + a_l) = e^{i 2 pi kappa_l} E(x) (P:L87,
Theorems "Periodicity along a1/a2/a3").  In grid units the
corrected lattice is the integer upper-triangular matrix Ag
(oracle.lattice), so the wrap is exact integer arithmetic: reduce the
neighbour by columns 3, 2, 1 of Ag (z, then y, then x) and multiply by
e^{i 2 pi kappa.t}.  Integer shifts preserve the Yee half offsets, so one
C_l serves every component.

Independent cross-check (``K1_paper``, ``K2_paper``, ``K3_paper``): the
paper's explicit block forms K1, K2 with the general J2
 and K3 with the four general J3 categories.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp


def _idx(a, b, c, n):
    return a + n[0] * (b + n[1] * c)


def shift(lat, kappa, axis):
    """Sparse S_axis: (S v)(r) = v(r + e_axis) with quasi-periodic wrap."""
    n = lat.n
    n1, n2, n3 = n
    Ag = lat.Ag
    c, b, a = np.meshgrid(np.arange(n3), np.arange(n2), np.arange(n1), indexing="ij")
    r = np.stack([a.ravel(), b.ravel(), c.ravel()], axis=0).astype(np.int64)
    rows = _idx(r[0], r[1], r[2], n)
    rp = r.copy()
    rp[axis] += 1
    t = np.zeros_like(rp)
    # z first, then y, then x (Ag upper triangular)
    for col, size in ((2, n3), (1, n2), (0, n1)):
        tc = np.floor_divide(rp[col], size)
        rp = rp - np.outer(Ag[:, col], tc)
        t[col] = tc
    phase = np.exp(2j * math.pi * (kappa[0] * t[0] + kappa[1] * t[1] + kappa[2] * t[2]))
    cols = _idx(rp[0], rp[1], rp[2], n)
    N = n1 * n2 * n3
    return sp.csr_matrix((phase, (rows, cols)), shape=(N, N))


def partials(lat, kappa):
    """C1, C2, C3."""
    N = lat.nn
    I = sp.identity(N, dtype=np.complex128, format="csr")
    return [((shift(lat, kappa, ax) - I) / lat.delta[ax]).tocsr() for ax in range(3)]


def curl(lat, kappa):
    """C = [[0,-C3,C2],[C3,0,-C1],[-C2,C1,0]]."""
    C1, C2, C3 = partials(lat, kappa)
    Z = sp.csr_matrix(C1.shape, dtype=np.complex128)
    return sp.bmat([[Z, -C3, C2], [C3, Z, -C1], [-C2, C1, Z]], format="csr")


def B_diag(eps_list):
    """B = diag(vec B1, vec B2, vec B3)."""
    return np.concatenate([np.ascontiguousarray(e, dtype=np.float64).ravel() for e in eps_list])


def dense_gep(lat, kappa, eps_list, null_rel=1e-10):
    """Plain definition: all eigenvalues of C*C e = lambda B e (P:L1642-1646,
    L2110-2112) by dense eigh of B^{-1/2} C*C B^{-1/2}.  Returns
    (all eigenvalues ascending, the nonzero ones, null count) with a
    null threshold null_rel * lambda_max."""
    C = curl(lat, kappa).toarray()
    A = C.conj().T @ C
    s = 1.0 / np.sqrt(B_diag(eps_list))
    H = (s[:, None] * A) * s[None, :]
    w = np.linalg.eigvalsh(H)
    thr = null_rel * max(1.0, abs(w[-1]))
    nz = w[np.abs(w) > thr]
    return w, nz, int(np.sum(np.abs(w) <= thr))


# ---------------------------------------------------------------------------
# The paper's explicit block forms (independent construction, for tests)
# ---------------------------------------------------------------------------

def _e(x):
    return np.exp(2j * math.pi * x)


def K1_paper(lat, kappa):
    """P:L896-902."""
    n1 = lat.n[0]
    K = -np.eye(n1, dtype=np.complex128) + np.eye(n1, k=1)
    K[n1 - 1, 0] += _e(kappa[0])
    return K / lat.delta[0]


def J2_paper(lat, kappa):
    """General J2 with rho1 from the snapping case."""
    n1 = lat.n[0]
    m1, rho1 = lat.m[0], lat.rho[0]
    J = np.zeros((n1, n1), dtype=np.complex128)
    J[:m1, n1 - m1:] = _e(-kappa[0]) * np.eye(m1)
    J[m1:, :n1 - m1] = np.eye(n1 - m1)
    return _e(rho1 * kappa[0]) * J


def K2_paper(lat, kappa):
    """K2 in C^{n1 n2}: block bidiagonal with corner e^{i2pi k.a2} J2."""
    n1, n2 = lat.n[0], lat.n[1]
    N = n1 * n2
    K = -np.eye(N, dtype=np.complex128)
    for j in range(n2 - 1):
        K[j * n1:(j + 1) * n1, (j + 1) * n1:(j + 2) * n1] += np.eye(n1)
    K[(n2 - 1) * n1:, :n1] += _e(kappa[1]) * J2_paper(lat, kappa)
    return K / lat.delta[1]


def _flags(lat):
    """rho4, rho5, psi1, psi2 of P:L763-775 from the corrected cosines."""
    cg, cb, ca = lat.cos
    n1 = lat.n[0]
    m1, m2, _ = lat.m
    r1, r2, r3 = lat.rho
    rho4 = int(math.ceil(cg * cb * (cg * cb - ca)))
    rho5 = int(math.ceil(cb))
    psi1 = 1 if ((r2 * n1 - m2) - (r1 * n1 - m1) > 0 and r3 == 0) else 0
    psi2 = 1 if ((r1 * n1 - m1) + (r2 * n1 - m2) > 0 and r3 == 1) else 0
    return rho4, rho5, psi1, psi2


def J3_category(lat):
    """The four general J3 categories."""
    n1 = lat.n[0]
    m1, m2, _ = lat.m
    if lat.rho[2] == 0:
        return 1 if m1 <= m2 else 2
    return 3 if m1 + m2 <= n1 else 4


def _perm_block(n1, top, phase_top):
    """[[0, phase_top I_top], [I_{n1-top}, 0]]"""
    J = np.zeros((n1, n1), dtype=np.complex128)
    J[:top, n1 - top:] = phase_top * np.eye(top)
    J[top:, :n1 - top] = np.eye(n1 - top)
    return J


def J3_paper(lat, kappa):
    """J3 of P:L776-844 (n1 n2 x n1 n2)."""
    n1, n2 = lat.n[0], lat.n[1]
    m1, m2, m3 = lat.m
    r1, r2, r3 = lat.rho
    rho4, rho5, psi1, psi2 = _flags(lat)
    k1, k2 = kappa[0], kappa[1]
    J1 = _e(r2 * k1) * _perm_block(n1, m2, _e(-k1))           # eq. (J1)
    cat = J3_category(lat)
    J = np.zeros((n1 * n2, n1 * n2), dtype=np.complex128)
    if cat in (1, 2):
        if cat == 1:
            ph = _e(-(k2 + r1 * rho4 * k1 - psi1 * k1))
            inner = _perm_block(n1, m2 - m1, _e(-k1))
        else:
            ph = _e(-(k2 - r2 * rho4 * k1 - psi1 * k1))
            inner = _perm_block(n1, n1 - m1 + m2, _e(-k1))
        top = ph * np.kron(np.eye(m3), inner)                 # rows 0..m3*n1
        bot = np.kron(np.eye(n2 - m3), J1)
        J[:m3 * n1, (n2 - m3) * n1:] = top
        J[m3 * n1:, :(n2 - m3) * n1] = bot
    else:
        top = _e(-k2) * np.kron(np.eye(m3), J1)
        if cat == 3:
            ph = _e((r1 * rho4 + psi2) * k1)
            inner = _perm_block(n1, m1 + m2, _e(-k1))
        else:
            ph = _e(-(rho5 * rho4 - psi2) * k1)
            inner = _perm_block(n1, m1 + m2 - n1, _e(-k1))
        bot = ph * np.kron(np.eye(n2 - m3), inner)
        J[:m3 * n1, (n2 - m3) * n1:] = top
        J[m3 * n1:, :(n2 - m3) * n1] = bot
    return _e(r3 * k2) * J


def K3_paper(lat, kappa):
    """K3 in C^{n}: block bidiagonal with corner e^{i2pi k.a3} J3."""
    n1, n2, n3 = lat.n
    P = n1 * n2
    N = P * n3
    K = -np.eye(N, dtype=np.complex128)
    for k in range(n3 - 1):
        K[k * P:(k + 1) * P, (k + 1) * P:(k + 2) * P] += np.eye(P)
    K[(n3 - 1) * P:, :P] += _e(kappa[2]) * J3_paper(lat, kappa)
    return K / lat.delta[2]
