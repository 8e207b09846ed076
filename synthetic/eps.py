"""Permittivity inputs sampled at Yee edge midpoints.

The Yee points of component l are x(a+1/2,b,c), x(a,b+1/2,c), x(a,b,c+1/2)
in the transformed Cartesian frame, i.e. ((a + h1) dx, (b + h2) dy,
(c + h3) dz) with h = e_l / 2.  The *geometry* (snapped lattice matrix and
spacings) is an argument computed by the caller; this module does not snap.
Shapes are defined in the ORIGINAL Cartesian frame: a Yee point is mapped to
fractional coordinates of the snapped cell and then to the original cell
(SURVEY.md B14/B19).  Point sampling, strict inequality (inside iff distance
< r).  Arrays are returned with shape (n3, n2, n1) (x fastest).

Recipes:
  sc_sphere       eps=13 in a sphere r=0.25 at the lattice points, else 1
  fcc_diamond     eps=13 rods r=0.11 from each lattice site to its 4 diamond
                  neighbours (a/4)(1,1,1),(1,-1,-1),(-1,1,-1),(-1,-1,1)
  bcc_sphere_rod  eps=13 spheres r=0.3 at lattice points + rods r=0.1 along
                  a1, a2, a3, a1+a2+a3 (the 4 nearest-neighbour bonds)
  gyroid[:<eps>]  eps (default 16) where the single-gyroid level set
                  sin(2 pi x/a) cos(2 pi y/a) + sin(2 pi y/a) cos(2 pi z/a)
                  + sin(2 pi z/a) cos(2 pi x/a) > 1.1, else 1 (PAPER.md
                  L2402-2407; BCC lattice; periodic under (a/2)(1,1,1))
  noise42         seed-42 Gaussian cell field smoothed (sigma=2 cells),
                  edge value = mean of its two endpoint cells, thresholded at
                  the median of the cell field -> eps in {1, 12}
  vacuum:<c>      constant eps = c (closed-form checks)
"""
from __future__ import annotations

import itertools

import numpy as np

EPS_IN = 13.0
EPS_OUT = 1.0


def yee_points(delta, n, comp):
    """Cartesian (transformed frame) coordinates of the Yee points of
    component ``comp`` (0,1,2), shape (n3*n2*n1, 3), x fastest."""
    n1, n2, n3 = n
    c, b, a = np.meshgrid(np.arange(n3), np.arange(n2), np.arange(n1), indexing="ij")
    idx = np.stack([a.ravel(), b.ravel(), c.ravel()], axis=1).astype(np.float64)
    idx[:, comp] += 0.5
    return idx * np.asarray(delta, dtype=np.float64)[None, :]


def _images(a_orig):
    ts = np.array(list(itertools.product((-1, 0, 1), repeat=3)), dtype=np.float64)
    return ts @ a_orig.T      # (27,3) lattice translations


def _seg_dist2(X, p0, p1):
    d = p1 - p0
    t = np.clip(((X - p0) @ d) / float(d @ d), 0.0, 1.0)
    r = X - (p0[None, :] + t[:, None] * d[None, :])
    return np.einsum("ij,ij->i", r, r)


def gyroid_level(X, a=1.0):
    """The gyroid level-set function of PAPER.md L2404-2405 at Cartesian points X (m, 3)."""
    u = 2.0 * np.pi * np.asarray(X, dtype=np.float64) / a
    return (np.sin(u[:, 0]) * np.cos(u[:, 1]) + np.sin(u[:, 1]) * np.cos(u[:, 2]) +
            np.sin(u[:, 2]) * np.cos(u[:, 0]))


def _inside(X, shape, a_orig):
    """X: (m,3) points in the original frame reduced into the primitive cell."""
    if shape == "gyroid":
        return gyroid_level(X) > 1.1
    imgs = _images(a_orig)
    inside = np.zeros(X.shape[0], dtype=bool)
    if shape == "sc_sphere":
        for s in imgs:
            inside |= np.einsum("ij,ij->i", X - s, X - s) < 0.25 ** 2
    elif shape == "fcc_diamond":
        bonds = 0.25 * np.array([[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]], dtype=np.float64)
        for s in imgs:
            for bd in bonds:
                inside |= _seg_dist2(X, s, s + bd) < 0.11 ** 2
    elif shape == "bcc_sphere_rod":
        bonds = [a_orig[:, 0], a_orig[:, 1], a_orig[:, 2], a_orig.sum(axis=1)]
        for s in imgs:
            inside |= np.einsum("ij,ij->i", X - s, X - s) < 0.3 ** 2
            for bd in bonds:
                inside |= _seg_dist2(X, s, s + bd) < 0.1 ** 2
    else:
        raise ValueError(shape)
    return inside


def _geometric(shape, a_snap, delta, n, a_orig, chunk=1 << 15, eps_in=EPS_IN):
    """Chunks of Yee points are independent, so they run on a thread pool (numpy releases the GIL in the
    distance kernels); every chunk computes exactly what the serial loop computed."""
    import concurrent.futures
    import os
    inv = np.linalg.inv(np.asarray(a_snap, dtype=np.float64))
    a_o = np.asarray(a_orig, dtype=np.float64)
    out = []
    workers = max(1, min(16, os.cpu_count() or 1))
    for comp in range(3):
        x = yee_points(delta, n, comp)
        e = np.empty(x.shape[0])

        def one(s, x=x, e=e):
            f = x[s:s + chunk] @ inv.T
            f -= np.floor(f)
            X = f @ a_o.T
            e[s:s + chunk] = np.where(_inside(X, shape, a_orig), eps_in, EPS_OUT)

        starts = range(0, x.shape[0], chunk)
        if workers > 1 and len(starts) > 1:
            with concurrent.futures.ThreadPoolExecutor(workers) as ex:
                list(ex.map(one, starts))
        else:
            for s in starts:
                one(s)
        out.append(e.reshape(n[2], n[1], n[0]))
    return out


def _noise(n, seed=42, sigma=2.0, lo=1.0, hi=12.0):
    n1, n2, n3 = n
    rng = np.random.default_rng(seed)
    f = rng.standard_normal((n3, n2, n1))
    fz, fy, fx = np.meshgrid(np.fft.fftfreq(n3), np.fft.fftfreq(n2), np.fft.fftfreq(n1), indexing="ij")
    filt = np.exp(-2.0 * np.pi ** 2 * sigma ** 2 * (fx ** 2 + fy ** 2 + fz ** 2))
    f = np.real(np.fft.ifftn(np.fft.fftn(f) * filt))
    med = np.median(f)
    out = []
    for axis in (2, 1, 0):               # component 1 varies along x (last numpy axis)
        e = 0.5 * (f + np.roll(f, -1, axis=axis))
        out.append(np.where(e > med, hi, lo).astype(np.float64))
    return out


def sample(shape, n, a_snap=None, delta=None, a_orig=None):
    """Return [eps1, eps2, eps3], each (n3, n2, n1) float64."""
    n = tuple(int(v) for v in n)
    if shape.startswith("vacuum"):
        c = float(shape.split(":")[1]) if ":" in shape else 1.0
        return [np.full((n[2], n[1], n[0]), c) for _ in range(3)]
    if shape == "noise42":
        return _noise(n)
    if shape.startswith("random"):
        # random:<seed>  i.i.d. eps in [1, 13) (stress input for parity tests)
        seed = int(shape.split(":")[1]) if ":" in shape else 0
        rng = np.random.default_rng(seed)
        return [1.0 + 12.0 * rng.random((n[2], n[1], n[0])) for _ in range(3)]
    if shape.startswith("gyroid"):
        eps_in = float(shape.split(":")[1]) if ":" in shape else 16.0
        return _geometric("gyroid", a_snap, delta, n, a_orig, eps_in=eps_in)
    return _geometric(shape, a_snap, delta, n, a_orig)


def stacked(eps_list):
    """Concatenate [eps1, eps2, eps3] into one (3*n,) float64 array."""
    return np.concatenate([np.ascontiguousarray(e).ravel() for e in eps_list])
