"""Fixture for the pure-C consumer of include/bnf.h (tests/c_abi/consumer.c):
a small FCC grid, seeded eps and vectors, and the oracle's dense A_r / M
applied to them.  Calls only oracle/ and synthetic/.

    python scripts/make_c_fixture.py   ->  tests/golden/c_abi_fcc654.bin

Layout (little endian): int32 n[3], int32 b, int32 op_count; float64 a_raw[9]
(column l = vector l, a_raw[3 l + r]); float64 kappa[3]; float64 eps[3n];
complex128 y[b][2n]; then for op in (A_r, M): complex128 want[b][2n].
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import lattice, spectral  # noqa: E402
from synthetic import configs, eps as E, vectors  # noqa: E402


def main():
    a = configs.fcc_vectors()
    n = (6, 5, 4)
    kap = (0.31, -0.12, 0.27)
    L = lattice.snap(a, n)
    eps = E.sample("fcc_diamond", n, L.a, L.delta, L.a_canon)
    b = 2
    y = vectors.complex_normal((b, 2 * L.nn), seed=77)
    out = os.path.join(ROOT, "tests", "golden", "c_abi_fcc654.bin")
    with open(out, "wb") as f:
        np.asarray(list(n) + [b, 2], dtype="<i4").tofile(f)
        np.ascontiguousarray(np.asarray(a, dtype="<f8").T).tofile(f)      # a_raw[3 l + r]
        np.asarray(kap, dtype="<f8").tofile(f)
        np.asarray(E.stacked(eps), dtype="<f8").tofile(f)
        np.asarray(y, dtype="<c16").tofile(f)
        for op in ("Ar", "M"):
            D = spectral.Ar_dense(L, kap, eps, op=op)
            np.asarray(y @ D.T, dtype="<c16").tofile(f)
    print(out)


if __name__ == "__main__":
    main()
