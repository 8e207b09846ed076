"""Eigensolver of the paper: inverse Lanczos on A_r with CG inner solves
(PAPER.md L2252-2260, L2398).  Test infrastructure only.

Per P:L2252-2255 each inverse-Lanczos step needs A_r^{-1} v
= Sigma_r^{-1} (Q_r^* B^{-1} Q_r)^{-1} Sigma_r^{-1} v, i.e. one CG solve with
the HPD operator M = Q_r^* B^{-1} Q_r (no preconditioner).
Readings: R12 tol_outer is the Ritz relative residual of
A_r^{-1}, |beta s_last| <= tol_outer |theta|;  R13 a block (b >= 1) Krylov
basis with full (twice, DGKS) reorthogonalisation and `guard` extra
converged pairs, because a single start vector cannot see a second copy of
a degenerate eigenvalue;  R6 Gamma-mode masking.
"""
from __future__ import annotations

import numpy as np


def cg(Mfun, c, tol=1e-13, maxit=2000):
    """Plain CG (Hestenes-Stiefel) for M x = c, column by column of c
    (shape (N,) or (N, b)); stops when ||r|| <= tol ||c||."""
    c = np.asarray(c)
    if c.ndim == 1:
        x, it = cg(Mfun, c[:, None], tol, maxit)
        return x[:, 0], it
    x = np.zeros_like(c)
    its = []
    for col in range(c.shape[1]):
        b = c[:, col]
        nb = np.linalg.norm(b)
        if nb == 0:
            its.append(0)
            continue
        xc = np.zeros_like(b)
        r = b.copy()
        p = r.copy()
        rr = np.vdot(r, r).real
        k = 0
        while np.sqrt(rr) > tol * nb and k < maxit:
            Mp = Mfun(p)
            alpha = rr / np.vdot(p, Mp).real
            xc += alpha * p
            r -= alpha * Mp
            rr_new = np.vdot(r, r).real
            p = r + (rr_new / rr) * p
            rr = rr_new
            k += 1
        x[:, col] = xc
        its.append(k)
    return x, its


def _orth(W, V_list):
    """Two rounds of classical Gram-Schmidt against all previous blocks (DGKS)."""
    for _ in range(2):
        for V in V_list:
            W = W - V @ (V.conj().T @ W)
    return W


def inverse_lanczos(op, nev, block=1, guard=0, tol_outer=1e-12, tol_inner=1e-13,
                    seed=0x5EED, max_steps=400):
    """Smallest nev eigenvalues of A_r (op: oracle.fftop.NFSEPOperator).
    Returns (lambda ascending (nev,), Ritz vectors (2n, nev), info dict)."""
    N = 2 * op.n
    sig = np.concatenate([op.sig.ravel(), op.sig.ravel()])
    mask = sig > 0
    sinv = np.where(mask, 1.0 / np.where(mask, sig, 1.0), 0.0)
    rng = np.random.default_rng(seed)
    V0 = (rng.standard_normal((N, block)) + 1j * rng.standard_normal((N, block))) * mask[:, None]
    V, _ = np.linalg.qr(V0)
    Vs = [V]
    Bs = []
    As = []
    inner = []
    want = nev + guard

    def opinv(X):
        Y, its = cg(op.M, sinv[:, None] * X, tol=tol_inner)
        inner.extend(its)
        return sinv[:, None] * Y

    theta = None
    for step in range(max_steps):
        W = opinv(Vs[-1])
        A = Vs[-1].conj().T @ W
        A = 0.5 * (A + A.conj().T)
        W = W - Vs[-1] @ A
        if Bs:
            W = W - Vs[-2] @ Bs[-1].conj().T
        W = _orth(W, Vs)
        Qn, R = np.linalg.qr(W)
        As.append(A)
        Bs.append(R)
        m = len(As)
        Tm = np.zeros((m * block, m * block), dtype=np.complex128)
        for s in range(m):
            Tm[s * block:(s + 1) * block, s * block:(s + 1) * block] = As[s]
            if s + 1 < m:
                Tm[(s + 1) * block:(s + 2) * block, s * block:(s + 1) * block] = Bs[s]
                Tm[s * block:(s + 1) * block, (s + 1) * block:(s + 2) * block] = Bs[s].conj().T
        theta, S = np.linalg.eigh(Tm)
        order = np.argsort(-theta)
        theta, S = theta[order], S[:, order]
        if m * block >= want:
            res = np.linalg.norm(R @ S[(m - 1) * block:, :want], axis=0)
            if np.all(res <= tol_outer * np.abs(theta[:want])):
                break
        Vs.append(Qn)
    Vall = np.concatenate(Vs[:len(As)], axis=1)
    Y = Vall @ S[:, :want]
    lam = 1.0 / theta[:want]
    o = np.argsort(lam)
    info = {"steps": len(As), "inner_iters": inner, "matvecs": int(np.sum(inner))}
    return lam[o][:nev], Y[:, o][:, :nev], info


def arpack_inverse(op, nev, guard=4, tol_outer=1e-12, tol_inner=1e-13, ncv=None,
                   seed=0x5EED):
    """Bounded-memory route to the same plain result (SURVEY.md §8(c) step
    5, "eigsh on a LinearOperator for A_r^{-1}"): the library implicitly
    restarted Lanczos (ARPACK, scipy.sparse.linalg.eigsh) on
    A_r^{-1} = Sigma_r^{-1} M^{-1} Sigma_r^{-1}, each
    application one CG solve with M to tol_inner, the Gamma mode
    masked (R6).  ARPACK's stopping test ||r_i|| <= tol |theta_i| on the
    Ritz pairs of A_r^{-1} is reading R12 with tol = tol_outer.  Used where
    the full Krylov basis of inverse_lanczos does not fit host memory
    (config 5, 256^3: one basis vector is 0.5 GiB).
    Returns (lambda ascending (nev,), Ritz vectors (2n, nev), info dict)."""
    from scipy.sparse.linalg import LinearOperator, eigsh

    N = 2 * op.n
    sig = np.concatenate([op.sig.ravel(), op.sig.ravel()])
    mask = sig > 0
    sinv = np.where(mask, 1.0 / np.where(mask, sig, 1.0), 0.0)
    inner = []

    def opinv(x):
        y, its = cg(op.M, sinv * np.ravel(x), tol=tol_inner)
        inner.extend(its)
        return sinv * y

    want = nev + guard
    rng = np.random.default_rng(seed)
    v0 = (rng.standard_normal(N) + 1j * rng.standard_normal(N)) * mask
    A = LinearOperator((N, N), matvec=opinv, dtype=np.complex128)
    theta, Y = eigsh(A, k=want, which="LA", v0=v0, tol=tol_outer,
                     ncv=ncv or max(2 * want + 1, 20), maxiter=10000)
    lam = 1.0 / theta
    o = np.argsort(lam)
    info = {"steps": len(inner), "inner_iters": inner, "matvecs": int(np.sum(inner))}
    return lam[o][:nev], Y[:, o][:, :nev], info
