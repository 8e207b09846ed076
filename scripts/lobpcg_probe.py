"""NEXT-1 decision probe (CPU, oracle operator): matvecs to the nev smallest
eigenvalues at 1e-10 relative accuracy by (a) the paper's inverse Lanczos with
CG inner solves (oracle.eigsolve.inverse_lanczos, block 2, guard 2) and (b)
LOBPCG on A_r preconditioned by Sigma_r^{-2} (scipy.sparse.linalg.lobpcg;
the preconditioned operator is similar to M, kappa <= max eps / min eps),
block nev + guard.  Config-4 lattice and eps at a reduced grid.

    python scripts/lobpcg_probe.py [n] [nev]
"""
import json
import os
import sys
import time

import numpy as np
from scipy.sparse.linalg import LinearOperator, lobpcg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import eigsolve, fftop, lattice  # noqa: E402
from synthetic import configs, eps as E  # noqa: E402


def main():
    n1 = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    nev = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    cfg = configs.config(4)
    n = (n1, n1, n1)
    L = lattice.snap(cfg.a_raw, n)
    eps = E.sample(cfg.shape, n, L.a, L.delta, L.a_canon)
    kap = lattice.kappa_from_raw(L, cfg.kappa_direct[7])
    op = fftop.NFSEPOperator(L, kap, eps)
    t = time.time()
    lam_l, _, info = eigsolve.inverse_lanczos(op, nev=nev, block=2, guard=2)
    t_l = time.time() - t
    N = 2 * op.n
    sig2 = np.concatenate([op.q.ravel(), op.q.ravel()])
    cnt = {"mv": 0}

    def mv(X):
        X = np.asarray(X)
        X2 = X.reshape(N, -1)
        cnt["mv"] += X2.shape[1]
        return np.stack([op.Ar(X2[:, j]) for j in range(X2.shape[1])], axis=1).reshape(X.shape)

    A = LinearOperator((N, N), matvec=mv, matmat=mv, dtype=np.complex128)
    T = LinearOperator((N, N), matvec=lambda x: np.ravel(x) / sig2, matmat=lambda X: X / sig2[:, None],
                       dtype=np.complex128)
    rng = np.random.default_rng(0)
    m = nev + 2
    X0 = rng.standard_normal((N, m)) + 1j * rng.standard_normal((N, m))
    t = time.time()
    lam_b, _, hist = lobpcg(A, X0, M=T, largest=False, tol=1e-7 * float(np.max(lam_l)), maxiter=2000,
                            retLambdaHistory=True)
    t_b = time.time() - t
    lam_b = np.sort(lam_b)[:nev]
    out = {"grid": n, "nev": nev, "inverse_lanczos_matvecs": int(info["matvecs"]), "inverse_lanczos_s": t_l,
           "lobpcg_iterations": len(hist), "lobpcg_matvecs": cnt["mv"], "lobpcg_s": t_b,
           "lobpcg_max_rel_dev": float(np.max(np.abs(lam_b - lam_l) / lam_l))}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
