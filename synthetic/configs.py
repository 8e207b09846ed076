"""The five workload configurations of BASELINE.json (made concrete in
SURVEY.md §8(d)).  Inputs only: raw lattice vectors (columns, Cartesian,
conventional constant a = 1), grid, Bloch vectors K (Cartesian, the physical
wave vector "2*pi*k" of PAPER.md L77-81), number of wanted eigenvalues.

The k-path convention follows PAPER.md L2398 ("segments connecting any two
corner points ... partition each segment"): corners are always included and
the interior points are distributed over segments in proportion to their
Cartesian length with largest-remainder rounding.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

TWO_PI = 2.0 * math.pi


@dataclass(frozen=True)
class Config:
    name: str
    a_raw: np.ndarray          # 3x3, columns are the primitive vectors (Cartesian)
    n: tuple                   # (n1, n2, n3)
    shape: str                 # permittivity recipe id (see synthetic.eps)
    nev: int
    kpoints: np.ndarray        # (K, 3) Cartesian Bloch vectors K = 2*pi*k
    labels: tuple = field(default_factory=tuple)
    kappa_direct: np.ndarray | None = None   # (K,3) reduced Bloch numbers, when the config gives them directly


def _cols(*v):
    return np.array(v, dtype=np.float64).T.copy()


def sc_vectors(a=1.0):
    return _cols([a, 0, 0], [0, a, 0], [0, 0, a])


def fcc_vectors(a=1.0):
    h = a / 2.0
    return _cols([0, h, h], [h, 0, h], [h, h, 0])


def bcc_vectors(a=1.0):
    h = a / 2.0
    return _cols([-h, h, h], [h, -h, h], [h, h, -h])


def triclinic_vectors(L1=1.0, L2=1.1, L3=1.2, alpha=80.0, beta=85.0, gamma=75.0):
    """Primitive vectors from lengths and angles (alpha = angle(a2,a3),
    beta = angle(a1,a3), gamma = angle(a1,a2)), built in the standard
    right-handed upper-triangular form."""
    ca, cb, cg = (math.cos(math.radians(t)) for t in (alpha, beta, gamma))
    sg = math.sin(math.radians(gamma))
    a1 = [L1, 0.0, 0.0]
    a2 = [L2 * cg, L2 * sg, 0.0]
    a3x = L3 * cb
    a3y = L3 * (ca - cb * cg) / sg
    a3z = math.sqrt(L3 * L3 - a3x * a3x - a3y * a3y)
    return _cols(a1, a2, [a3x, a3y, a3z])


def path_points(corners: dict, labels: list, total: int):
    """Points along the polyline through ``labels``: all corners plus
    ``total - len(labels)`` interior points, split over segments by length
    (largest remainder), evenly spaced inside each segment."""
    P = [np.asarray(corners[l], dtype=np.float64) for l in labels]
    seg = [float(np.linalg.norm(P[i + 1] - P[i])) for i in range(len(P) - 1)]
    interior = total - len(P)
    share = [interior * s / sum(seg) for s in seg]
    cnt = [int(math.floor(x)) for x in share]
    rem = interior - sum(cnt)
    order = sorted(range(len(seg)), key=lambda i: (-(share[i] - cnt[i]), i))
    for i in order[:rem]:
        cnt[i] += 1
    pts, lab = [P[0]], [labels[0]]
    for s in range(len(seg)):
        m = cnt[s]
        for q in range(1, m + 1):
            t = q / (m + 1)
            pts.append((1 - t) * P[s] + t * P[s + 1])
            lab.append("")
        pts.append(P[s + 1])
        lab.append(labels[s + 1])
    return np.array(pts), tuple(lab), tuple(cnt)


# Standard FCC Brillouin-zone corners (units 2*pi/a); the paper's appendix
# table is absent from PAPER.md (L240), see SURVEY.md B13.
FCC_CORNERS = {
    "G": (0.0, 0.0, 0.0), "X": (0.0, 1.0, 0.0), "U": (0.25, 1.0, 0.25),
    "L": (0.5, 0.5, 0.5), "W": (0.5, 1.0, 0.0), "K": (0.75, 0.75, 0.0),
}
# BCC corners printed in PAPER.md L270-283 (units 2*pi/a).
BCC_CORNERS = {
    "G": (0.0, 0.0, 0.0), "H": (0.0, 1.0, 0.0), "N": (0.5, 0.5, 0.0),
    "P": (0.5, 0.5, 0.5),
}


def _scaled(corners, s):
    return {k: tuple(s * x for x in v) for k, v in corners.items()}


def config(idx: int) -> Config:
    """BASELINE.json configs[idx-1] (1-based)."""
    if idx == 1:
        K = np.array([[math.pi * 0.5, math.pi * 0.3, math.pi * 0.1]])
        return Config("sc12_sphere", sc_vectors(), (12, 12, 12), "sc_sphere", 10, K, ("k1",))
    if idx == 2:
        pts, lab, _ = path_points(_scaled(FCC_CORNERS, TWO_PI), list("XULGXWK"), 40)
        return Config("fcc64_diamond", fcc_vectors(), (64, 64, 64), "fcc_diamond", 10, pts, lab)
    if idx == 3:
        pts, lab, _ = path_points(_scaled(BCC_CORNERS, TWO_PI), list("GHNGPH"), 30)
        return Config("bcc96_spheres_rods", bcc_vectors(), (96, 96, 96), "bcc_sphere_rod", 12, pts, lab)
    if idx == 4:
        kap = np.array([[t / 23 * 0.5] * 3 for t in range(24)])
        return Config("triclinic128_noise", triclinic_vectors(), (128, 128, 128), "noise42", 16,
                      np.zeros((24, 3)), tuple(["G"] + [""] * 22 + ["R"]), kappa_direct=kap)
    if idx == 5:
        K = np.array([[math.pi * 1.0, math.pi * 0.5, 0.0]])
        return Config("fcc256_diamond", fcc_vectors(), (256, 256, 256), "fcc_diamond", 10, K, ("k5",))
    raise ValueError(idx)


def with_grid(cfg: Config, n) -> Config:
    """Same lattice/shape/k-set on another grid (smaller parity cases)."""
    return Config(cfg.name + "_%dx%dx%d" % tuple(n), cfg.a_raw, tuple(n), cfg.shape, cfg.nev,
                  cfg.kpoints, cfg.labels, cfg.kappa_direct)
