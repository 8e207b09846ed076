"""Oracle eigenvalues at FULL BASELINE grids on k-subsets (slow: numpy
matrix-free A_r + the oracle's inverse Lanczos).  Calls only oracle/ and
synthetic/.  Writes tests/golden/full_<config>_<k>_oracle.json.

    python scripts/make_golden_full.py [--route lanczos|arpack] <config> <k_index> [<k_index> ...]

Route "lanczos" (default): oracle.eigsolve.inverse_lanczos, block 4, guard 4.
Route "arpack": oracle.eigsolve.arpack_inverse (bounded memory; 256^3).
Set ORACLE_THREADS / ORACLE_FFT_WORKERS to use several host cores (execution
only: the operator result is bit-identical, tests/test_oracle_solver.py).
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import eigsolve, fftop, lattice  # noqa: E402
from synthetic import configs, eps as E  # noqa: E402


def main():
    argv = sys.argv[1:]
    route = "lanczos"
    if argv[0] == "--route":
        route, argv = argv[1], argv[2:]
    idx = int(argv[0])
    cfg = configs.config(idx)
    L = lattice.snap(cfg.a_raw, cfg.n)
    eps = E.sample(cfg.shape, cfg.n, L.a, L.delta, L.a_canon)
    h = hashlib.sha256(np.concatenate([np.ravel(e) for e in eps]).tobytes()).hexdigest()[:16]
    for kidx in (int(x) for x in argv[1:]):
        if cfg.kappa_direct is not None:
            kap = lattice.kappa_from_raw(L, cfg.kappa_direct[kidx])
        else:
            kap = lattice.kvec_reduce(L, cfg.kpoints[kidx])
        op = fftop.NFSEPOperator(L, kap, eps)
        t = time.time()
        if route == "arpack":
            lam, Y, info = eigsolve.arpack_inverse(op, nev=cfg.nev, guard=4)
            src = "oracle.eigsolve.arpack_inverse (SURVEY 8(c) step 5; ARPACK on A_r^{-1}, guard 4, "
        else:
            lam, Y, info = eigsolve.inverse_lanczos(op, nev=cfg.nev, block=4, guard=4)
            src = "oracle.eigsolve.inverse_lanczos (P:L2252-2260, L2398; block 4, guard 4, "
        res = [float(np.linalg.norm(op.Ar(Y[:, i]) - lam[i] * Y[:, i]) / np.linalg.norm(Y[:, i]))
               for i in range(cfg.nev)]
        out = {"_source": "scripts/make_golden_full.py: " + src + "tol 1e-12/1e-13) on oracle.fftop.NFSEPOperator",
               "config": idx, "name": cfg.name, "n": list(cfg.n), "k_index": kidx, "kappa": list(kap),
               "eps_sha256_16": h, "lambda": [float(x) for x in lam], "residuals": res,
               "steps": info["steps"], "matvecs": info["matvecs"], "seconds": time.time() - t}
        path = os.path.join(ROOT, "tests", "golden", "full_c%d_k%d_oracle.json" % (idx, kidx))
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
        print(path, out["seconds"], flush=True)


if __name__ == "__main__":
    main()
