"""Matrix-free null-space-free operator: PAPER.md §5.3 (L2264-2391),
Algorithms 1 (T^* p) and 2 (T q), with numpy FFTs as the DFT primitive.
Test infrastructure only.

Arrays are (n3, n2, n1) = [k or c, j or b, i or a] (x fastest), the same
layout as oracle.spectral.  U_n is the un-normalised inverse
DFT matrix U[s, t] = e^{+2 pi i s t / n}:  U x = n * ifft(x),
U^* x = fft(x).  Normalisation: T is unitary with n^{-1/2}
(eq. T); the "1/n" printed in the algorithms is
read as n^{-1/2} each way (R7b).

Execution knobs (no effect on the arithmetic): ORACLE_FFT_WORKERS (default
1) is passed to scipy.fft as `workers` (threads over independent 1D
transforms); ORACLE_THREADS (default 1) > 1 runs the three components of
M / recover in threads.  Each component's chain is unchanged and the
component contributions are summed in the fixed order l = 0, 1, 2, so the
result is bit-identical to the serial loop.
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.fft as _sfft

from . import spectral

_WORKERS = int(os.environ.get("ORACLE_FFT_WORKERS", "1"))
_THREADS = int(os.environ.get("ORACLE_THREADS", "1"))


def _ifft(x, axis):
    return _sfft.ifft(x, axis=axis, workers=_WORKERS)


def _fft(x, axis):
    return _sfft.fft(x, axis=axis, workers=_WORKERS)


def _per_component(fn):
    """[fn(0), fn(1), fn(2)], serially or in threads (independent chains)."""
    if _THREADS > 1:
        with ThreadPoolExecutor(3) as ex:
            return list(ex.map(fn, range(3)))
    return [fn(l) for l in range(3)]


def _diag_phases(lat, kappa):
    """D_{a1}, D_{a^2,i}, D_{a^3,i,j} (eq. diagonal_matrix) as
    broadcastable arrays over (c, b, a) / (c, j, i)."""
    n1, n2, n3 = lat.n
    m1, m2, m3 = lat.m
    kh2, kh3 = spectral.kappa_hat(lat, kappa)
    i = np.arange(n1)[None, None, :]
    j = np.arange(n2)[None, :, None]
    a = np.arange(n1)[None, None, :]
    b = np.arange(n2)[None, :, None]
    c = np.arange(n3)[:, None, None]
    if lat.rho[2] == 0:
        coef = -((n2 - m3) / n2) * (m1 / n1) + (m1 - m2) / n1
    else:
        coef = -((n2 - m3) / n2) * (m1 / n1) - m2 / n1
    th_a3 = 2 * math.pi * (kh3 - (m3 / n2) * j + coef * i) / n3      # theta_{a^3,i,j}
    th_a2 = 2 * math.pi * (kh2 - (m1 / n1) * i) / n2                 # theta_{a^2,i}
    th_a1 = 2 * math.pi * kappa[0] / n1                              # theta_{a1}
    D3 = np.exp(1j * c * th_a3)      # (n3, n2, n1): over (c, j, i)
    D2 = np.exp(1j * b * th_a2)      # (1, n2, n1):  over (b, i)
    D1 = np.exp(1j * a * th_a1)      # (1, 1, n1):   over a
    return D1, D2, D3


def T_apply(lat, kappa, q, D=None):
    """Algorithm 2: T q."""
    n1, n2, n3 = lat.n
    D1, D2, D3 = D or _diag_phases(lat, kappa)
    x = _ifft(q, axis=0) * n3          # U_n3 along k -> c
    x = x * D3                               # D_{a^3,i,j}
    x = _ifft(x, axis=1) * n2          # U_n2 along j -> b
    x = x * D2                               # D_{a^2,i}
    x = _ifft(x, axis=2) * n1          # U_n1 along i -> a
    x = x * D1                               # D_{a1}
    return x / math.sqrt(n1 * n2 * n3)


def Tstar_apply(lat, kappa, p, D=None):
    """Algorithm 1: T^* p (exact adjoint of Algorithm 2)."""
    n1, n2, n3 = lat.n
    D1, D2, D3 = D or _diag_phases(lat, kappa)
    x = p * np.conj(D1)
    x = _fft(x, axis=2)
    x = x * np.conj(D2)
    x = _fft(x, axis=1)
    x = x * np.conj(D3)
    x = _fft(x, axis=0)
    return x / math.sqrt(n1 * n2 * n3)


class NFSEPOperator:
    """y in C^{2n} (y1, y2 in Fourier layout) -> A_r y or M y.
    M = Q_r^* B^{-1} Q_r is the CG operator; A_r = Sigma_r M Sigma_r."""

    def __init__(self, lat, kappa, eps_list):
        self.lat = lat
        self.kappa = tuple(float(k) for k in kappa)
        self.n = lat.nn
        shp = (lat.n[2], lat.n[1], lat.n[0])
        _, Pi1, Pi2, q = spectral.pis(lat, kappa)
        self.Pi1 = Pi1.reshape((3,) + shp)
        self.Pi2 = Pi2.reshape((3,) + shp)
        self.q = q.reshape(shp)
        self.sig = np.sqrt(self.q)
        self.binv = [1.0 / np.asarray(e, dtype=np.float64).reshape(shp) for e in eps_list]
        self.D = _diag_phases(lat, kappa)
        self.shp = shp
        self.mask = (self.q > 0).astype(np.float64)

    def M(self, y):
        n = self.n
        y = np.asarray(y).reshape(2, *self.shp)

        def comp(l):
            v = self.Pi1[l] * y[0] + self.Pi2[l] * y[1]          # Q_r y, Fourier side
            u = T_apply(self.lat, self.kappa, v, self.D)        # real space
            w = Tstar_apply(self.lat, self.kappa, u * self.binv[l], self.D)
            return np.conj(self.Pi1[l]) * w, np.conj(self.Pi2[l]) * w

        z1 = np.zeros(self.shp, dtype=np.complex128)
        z2 = np.zeros(self.shp, dtype=np.complex128)
        for c1, c2 in _per_component(comp):
            z1 += c1
            z2 += c2
        return np.concatenate([z1.ravel(), z2.ravel()])

    def Ar(self, y):
        s = np.concatenate([self.sig.ravel(), self.sig.ravel()])
        return s * self.M(s * np.asarray(y).ravel())

    def apply(self, y, op="Ar"):
        return self.Ar(y) if op == "Ar" else self.M(y)

    def recover(self, y):
        """e = B^{-1} Q_r Sigma_r y, real-space Yee layout
        (3, n3, n2, n1)."""
        y = np.asarray(y).reshape(2, *self.shp)

        def comp(l):
            v = self.sig * (self.Pi1[l] * y[0] + self.Pi2[l] * y[1])
            return T_apply(self.lat, self.kappa, v, self.D) * self.binv[l]

        return np.stack(_per_component(comp))
