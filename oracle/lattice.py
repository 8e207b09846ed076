"""Lattice geometry: PAPER.md §2.2-2.3 (L131-283).  Test infrastructure only.

Conventions (DESIGN.md "Readings" R10, R11):
* Input: three primitive vectors a~_1..3 as the COLUMNS of a 3x3 matrix in
  any Cartesian frame.
* Canonicalisation (P:L143 requires |a1| >= |a2|, |a3|): cyclic relabel so
  the longest vector comes first (ties -> lowest index); if the relabelled
  triple is left-handed, negate a3.
* Angles: gamma = angle(a1,a2), beta = angle(a1,a3), alpha = angle(a2,a3).
* Snapping rounds "half up": fraction < 1/2 -> floor, otherwise ceil
  (the two half-open conditions of P:L151-152 etc.).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


class GeometryError(ValueError):
    pass


@dataclass
class Lattice:
    n: tuple            # (n1, n2, n3)
    perm: tuple         # canonical vector l = raw vector perm[l]
    sign3: int          # +1, or -1 if a3 was negated
    a_canon: np.ndarray # canonical raw vectors (columns), original frame
    lengths: tuple      # |a1|, |a2|, |a3|
    cos_raw: tuple      # (cos gamma', cos beta', cos alpha')
    m: tuple            # (m1, m2, m3)
    rho: tuple          # (rho1, rho2, rho3)
    cos: tuple          # corrected (cos gamma, cos beta, cos alpha)
    a: np.ndarray       # eq. (transvec): corrected vectors, columns, upper triangular
    l: tuple            # (l1, l2, l3)
    delta: tuple        # (dx, dy, dz)
    Ag: np.ndarray      # integer lattice in grid units: a = diag(delta) @ Ag

    @property
    def nn(self):
        return self.n[0] * self.n[1] * self.n[2]


def _round_half_up(q):
    """floor if 0 <= q - floor(q) < 1/2, ceil otherwise."""
    f = math.floor(q)
    return int(f) if q - f < 0.5 else int(f) + 1


def canonicalize(a_raw):
    a_raw = np.asarray(a_raw, dtype=np.float64)
    L = [float(np.linalg.norm(a_raw[:, i])) for i in range(3)]
    p = max(range(3), key=lambda i: (L[i], -i))   # longest, ties -> lowest index
    perm = (p, (p + 1) % 3, (p + 2) % 3)
    a = a_raw[:, list(perm)].copy()
    sign3 = 1
    if np.linalg.det(a) < 0:
        a[:, 2] = -a[:, 2]
        sign3 = -1
    return a, perm, sign3


def snap(a_raw, n):
    """PAPER.md §2.2: isometric frame, angle snapping Cases I/II
    for m1, m2, m3, corrected vectors
    eq. (transvec)."""
    n1, n2, n3 = (int(v) for v in n)
    if min(n1, n2, n3) < 1:
        raise ValueError("grid sizes must be positive")
    a, perm, sign3 = canonicalize(a_raw)
    L1, L2, L3 = (float(np.linalg.norm(a[:, i])) for i in range(3))
    cg_r = float(a[:, 0] @ a[:, 1]) / (L1 * L2)
    cb_r = float(a[:, 0] @ a[:, 2]) / (L1 * L3)
    ca_r = float(a[:, 1] @ a[:, 2]) / (L2 * L3)
    sg_r = math.sqrt(max(0.0, 1.0 - cg_r * cg_r))
    # P:L143 admissibility (with the raw angles)
    if not (L1 >= L2 and L1 >= L3):
        raise GeometryError("P:L143 |a1| >= |a2|,|a3| violated")
    if not (L2 * sg_r > L3 * abs(ca_r - cg_r * cb_r) / sg_r):
        raise GeometryError("P:L143 |a2| sin(gamma) > |a3||cos(alpha)-cos(gamma)cos(beta)|/sin(gamma) violated")

    dx = L1 / n1
    # --- gamma -> m1
    if cg_r >= 0.0:                                  # Case I: 0 < gamma' <= pi/2
        m1 = _round_half_up(L2 * cg_r / dx)
        cg = m1 * dx / L2
        rho1 = 0
    else:                                            # Case II
        m1 = _round_half_up((L1 + L2 * cg_r) / dx)
        cg = (m1 * dx - L1) / L2
        rho1 = 1
    if abs(cg) >= 1.0:
        raise GeometryError("|cos gamma| >= 1 after snapping")
    sg = math.sqrt(1.0 - cg * cg)
    l2 = L2 * sg
    dy = l2 / n2
    # --- beta -> m2
    if cb_r >= 0.0:
        m2 = _round_half_up(L3 * cb_r / dx)
        cb = m2 * dx / L3
        rho2 = 0
    else:
        m2 = _round_half_up((L1 + L3 * cb_r) / dx)
        cb = (m2 * dx - L1) / L3
        rho2 = 1
    if abs(cb) >= 1.0:
        raise GeometryError("|cos beta| >= 1 after snapping")
    # --- alpha -> m3; Case I also takes D' = 0 (m3 = 0)
    D = ca_r - cg * cb
    if D >= 0.0:
        m3 = _round_half_up(L3 * D / (dy * sg))
        ca = m3 * dy * sg / L3 + cg * cb
        rho3 = 0
    else:
        m3 = _round_half_up((L2 * sg * sg + L3 * D) / (dy * sg))
        ca = (m3 * dy * sg - L2 * sg * sg) / L3 + cg * cb
        rho3 = 1
    if not (0 <= m1 <= n1 and 0 <= m2 <= n1 and 0 <= m3 <= n2):
        raise GeometryError("snapped m outside 0<=m1,m2<=n1, 0<=m3<=n2 (P:L148-201)")
    vol = 1.0 - cg * cg - cb * cb - ca * ca + 2.0 * cg * cb * ca
    if not vol > 0.0:
        raise GeometryError("degenerate cell after snapping")
    # eq. (transvec)
    A = np.array([[L1, L2 * cg, L3 * cb],
                  [0.0, L2 * sg, L3 * (ca - cg * cb) / sg],
                  [0.0, 0.0, L3 * math.sqrt(vol) / sg]])
    l1, l3 = L1, float(A[2, 2])
    delta = (dx, dy, l3 / n3)
    Ag = np.array([[n1, m1 - rho1 * n1, m2 - rho2 * n1],
                   [0, n2, m3 - rho3 * n2],
                   [0, 0, n3]], dtype=np.int64)
    return Lattice((n1, n2, n3), perm, sign3, a, (L1, L2, L3), (cg_r, cb_r, ca_r),
                   (m1, m2, m3), (rho1, rho2, rho3), (cg, cb, ca), A, (l1, l2, l3), delta, Ag)


def kvec_reduce(lat: Lattice, K_cart):
    """Reduced Bloch numbers kappa_l = k . a_l with 2*pi*k = K:
    kappa_l = K . a~_l / (2 pi), a~ the canonical raw vectors.  Invariant
    under the isometry and Omega."""
    K = np.asarray(K_cart, dtype=np.float64)
    return tuple(float(K @ lat.a_canon[:, l]) / (2.0 * math.pi) for l in range(3))


def kappa_from_raw(lat: Lattice, kappa_raw):
    """Reorder reduced Bloch numbers given w.r.t. the raw labelling into the
    canonical labelling (and flip kappa3 if a3 was negated)."""
    k = [float(kappa_raw[lat.perm[l]]) for l in range(3)]
    k[2] *= lat.sign3
    return tuple(k)


def reciprocal(lat: Lattice):
    """b = 2 pi a^{-T};  Omega = a^{-T} a~^T."""
    b = 2.0 * math.pi * np.linalg.inv(lat.a).T
    omega = np.linalg.inv(lat.a).T @ lat.a_canon.T
    return b, omega
