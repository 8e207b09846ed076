"""Closed-form spectral decomposition and the dense null-space-free operator:
PAPER.md §4 (L1649-2104) and §5.1-5.2 (L2108-2262).  Test infrastructure
only.

Fourier (column) index of T: (i, j, k), stored x-fastest
col = i + n1*(j + n2*k).  The paper orders T's columns with i slowest
(P:L2008-2025); that is a column permutation of the same unitary T and does
not change any spectrum (R9).

Readings:
  R1  theta_{i,j,k} branch: coefficient (m1 m3 - n2 m2)/(n1 n2) when
      cos(alpha) - cos(beta)cos(gamma) >= 0 (Thm eigK3_acute),
      (m1 m3 - n2 m1 - n2 m2)/(n1 n2) otherwise (Thm eigK3_obtuse,
      P:L1864-1872); the conditions printed at P:L2035/L2041 are swapped.
  R2  Lambda_s = Lambda1+Lambda2+Lambda3;  Lambda_p = [L3-L2; L1-L3; L2-L1]
      (3n x n), so Lambda_p^* Lambda_p = sum of |pairwise differences|^2
      (P:L2125 as printed is inconsistent with its use at P:L2171-2188).
  R3  Pi1 = [Lq - L1 Ls^*; Lq - L2 Ls^*; Lq - L3 Ls^*] (Lp^*Lp Lq)^{-1/2}
      (P:L2172-2176).
  R4  The NFSEP uses Q_r, not P_r (BASELINE north_star wording).
  R5  Where Lambda_p^*Lambda_p <= TAU_P * Lambda_q for a mode (P:L2128's
      full-rank claim fails, e.g. lambda1=lambda2=lambda3), Pi1/Pi2 are
      replaced by: e_m with the smallest |lambda_m| (ties -> lowest m)
      Gram-Schmidt'ed against Pi0, and conj(Pi0 x Pi1').
  R6  Gamma (all kappa integer, P:L2221 defers): the single mode with
      g = 0 mod 1 has Lambda_q = 0; Pi0, Pi1, Pi2 and Sigma_r are set to 0
      there.
  R7  e^{theta} - 1 evaluated as 2i sin(theta/2) e^{theta/2} (exact
      identity; avoids cancellation for small theta).
"""
from __future__ import annotations

import math

import numpy as np

TAU_P = 1e-6


def kappa_hat(lat, kappa):
    """kappa.a^_2 (Thm eigK2) and kappa.a^_3 (Thm eigK3_acute
    P:L1733 / eigK3_obtuse P:L1872)."""
    n1, n2, _ = lat.n
    m1, m2, m3 = lat.m
    r1, r2, r3 = lat.rho
    k1, k2, k3 = kappa
    kh2 = k2 - (m1 / n1) * k1 + r1 * k1
    if r3 == 0:   # acute (R1)
        kh3 = (k3 - (m3 / n2) * k2 - ((n2 - m3) / n2) * (m1 / n1) * k1 + ((m1 - m2) / n1) * k1
               + r3 * k2 - (m3 / n2) * r1 * k1 + r2 * k1)
    else:         # obtuse
        kh3 = (k3 - (m3 / n2) * k2 - ((n2 - m3) / n2) * (m1 / n1) * k1 - (m2 / n1) * k1
               + r3 * k2 - (m3 / n2) * r1 * k1 + r1 * k1 + r2 * k1)
    return kh2, kh3


def thetas(lat, kappa):
    """theta_i, theta_{i,j}, theta_{i,j,k} / i  (real phases, radians) as
    arrays broadcast over (k, j, i) -> shape (n3, n2, n1)."""
    n1, n2, n3 = lat.n
    m1, m2, m3 = lat.m
    kh2, kh3 = kappa_hat(lat, kappa)
    kk, jj, ii = np.meshgrid(np.arange(n3), np.arange(n2), np.arange(n1), indexing="ij")
    th1 = 2 * math.pi * (ii + kappa[0]) / n1                                  # (eq. ewK1)
    th2 = 2 * math.pi * (jj - (m1 / n1) * ii + kh2) / n2                      # (eq. ewK2)
    if lat.rho[2] == 0:
        coef = -((n2 - m3) / n2) * (m1 / n1) + (m1 - m2) / n1                 # (eq. acute_ewK3)
    else:
        coef = -((n2 - m3) / n2) * (m1 / n1) - m2 / n1                        # (eq. obtuse_ewK3)
    th3 = 2 * math.pi * (kk - (m3 / n2) * jj + coef * ii + kh3) / n3
    return th1, th2, th3


def _em1(th):
    """e^{i th} - 1 = 2i sin(th/2) e^{i th/2}  (R7)."""
    return 2j * np.sin(0.5 * th) * np.exp(0.5j * th)


def lambdas(lat, kappa):
    """Lambda_1, Lambda_2, Lambda_3 diagonals, each (n3,n2,n1)."""
    th1, th2, th3 = thetas(lat, kappa)
    dx, dy, dz = lat.delta
    return _em1(th1) / dx, _em1(th2) / dy, _em1(th3) / dz


def gamma_mode(lat, kappa):
    """Flat index of the g = 0 mode when every kappa_l is an integer (R6),
    else None.  Exact rational test on the theta numerators."""
    if not all(float(k).is_integer() for k in kappa):
        return None
    th1, th2, th3 = thetas(lat, kappa)
    n1, n2, n3 = lat.n
    # theta/(2 pi) * n_l is integral for integer kappa: test with rounding
    r = [np.abs(t / (2 * math.pi) - np.round(t / (2 * math.pi))) for t in (th1, th2, th3)]
    hit = np.flatnonzero(((r[0] < 1e-9) & (r[1] < 1e-9) & (r[2] < 1e-9)).ravel())
    assert hit.size == 1, hit
    return int(hit[0])


def pis(lat, kappa):
    """Per-mode Pi0, Pi1, Pi2 (3 x n each, P:L2129-2192 with R2/R3/R5/R6) and
    Lambda_q (n,).  Component l of Pi_c is row l."""
    L1, L2, L3 = (x.ravel() for x in lambdas(lat, kappa))
    lam = np.stack([L1, L2, L3])                    # 3 x n
    q = np.sum(np.abs(lam) ** 2, axis=0)            # Lambda_q
    ls = L1 + L2 + L3                               # Lambda_s
    lp = np.stack([L3 - L2, L1 - L3, L2 - L1])      # Lambda_p (R2)
    p2 = np.sum(np.abs(lp) ** 2, axis=0)            # Lambda_p^* Lambda_p
    g = gamma_mode(lat, kappa)
    good = q > 0
    if g is not None:
        good[g] = False
    qs = np.where(good, q, 1.0)
    Pi0 = np.where(good, lam / np.sqrt(qs), 0)                          # (eq. null_basis)
    ok = good & (p2 > TAU_P * q)
    p2s = np.where(ok, p2, 1.0)
    Pi1 = np.where(ok, (q[None, :] - lam * np.conj(ls)[None, :]) / np.sqrt(p2s * qs), 0)   # R3
    Pi2 = np.where(ok, np.conj(lp) / np.sqrt(p2s), 0)                   # (eq. range_basis2)
    for idx in np.flatnonzero(good & ~ok):                              # R5 fallback
        u = Pi0[:, idx]
        m = int(np.argmin(np.abs(lam[:, idx])))
        e = np.zeros(3, dtype=np.complex128)
        e[m] = 1.0
        v = e - u * np.conj(u[m])
        v = v / np.linalg.norm(v)
        w = np.conj(np.cross(u, v))
        Pi1[:, idx] = v
        Pi2[:, idx] = w
    return Pi0, Pi1, Pi2, np.where(good, q, 0.0)


def T_dense(lat, kappa):
    """T = n^{-1/2} [z_{ijk} (x) y_{ij} (x) x_i]  (eq. T),
    entries T[(a,b,c),(i,j,k)] = n^{-1/2} e^{a th_i + b th_ij + c th_ijk}."""
    n1, n2, n3 = lat.n
    th1, th2, th3 = (t.ravel() for t in thetas(lat, kappa))
    cc, bb, aa = np.meshgrid(np.arange(n3), np.arange(n2), np.arange(n1), indexing="ij")
    a, b, c = aa.ravel(), bb.ravel(), cc.ravel()
    ph = np.outer(a, th1) + np.outer(b, th2) + np.outer(c, th3)
    return np.exp(1j * ph) / math.sqrt(n1 * n2 * n3)


def Q_dense(lat, kappa):
    """Q = (I3 (x) T)[Pi1 Pi2 Pi0]; returns (Q0, Q1, Q2)."""
    T = T_dense(lat, kappa)
    Pi0, Pi1, Pi2, _ = pis(lat, kappa)
    f = lambda P: np.concatenate([T * P[l][None, :] for l in range(3)], axis=0)
    return f(Pi0), f(Pi1), f(Pi2)


def P_dense(lat, kappa):
    """P = (I3 (x) T)[-conj(Pi2), conj(Pi1), conj(Pi0)];
    returns (P0, P1, P2) with P1 = conj-Pi1 and P2 = -conj-Pi2 columns."""
    T = T_dense(lat, kappa)
    Pi0, Pi1, Pi2, _ = pis(lat, kappa)
    f = lambda P: np.concatenate([T * P[l][None, :] for l in range(3)], axis=0)
    return f(np.conj(Pi0)), f(np.conj(Pi1)), f(-np.conj(Pi2))


def Ar_dense(lat, kappa, eps_list, op="Ar"):
    """A_r = Sigma_r Q_r^* B^{-1} Q_r Sigma_r  (NFSEP) with
    Q_r = [Q1, Q2], Sigma_r = diag(Lq^{1/2}, Lq^{1/2}).
    op="M" returns Q_r^* B^{-1} Q_r (the CG operator).
    2n x 2n, y = [y1; y2] with y1, y2 in the Fourier layout."""
    _, Q1, Q2 = Q_dense(lat, kappa)
    Qr = np.concatenate([Q1, Q2], axis=1)
    binv = 1.0 / np.concatenate([np.ravel(e) for e in eps_list])
    M = Qr.conj().T @ (binv[:, None] * Qr)
    if op == "M":
        return M
    _, _, _, q = pis(lat, kappa)
    s = np.sqrt(np.concatenate([q, q]))
    return (s[:, None] * M) * s[None, :]


def free_photon(lat, kappa, c=1.0):
    """Closed form for eps == c: A_r = Sigma_r^2 / c, eigenvalues
    Lambda_q / c (each twice) with Lambda_q = sum_l 4 sin^2(theta_l/2)/delta_l^2."""
    th1, th2, th3 = thetas(lat, kappa)
    q = sum(4.0 * np.sin(0.5 * t) ** 2 / d ** 2 for t, d in zip((th1, th2, th3), lat.delta))
    return np.sort(np.concatenate([q.ravel(), q.ravel()]) / c)
