"""Writes tests/golden/*_oracle.json.  Calls only oracle/ (and synthetic/ for
inputs) -- never the CUDA path.  Usage: python scripts/make_golden.py"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import curl, lattice, spectral  # noqa: E402
from synthetic import configs, eps as E  # noqa: E402


def eps_hash(eps):
    return hashlib.sha256(np.concatenate([np.ravel(e) for e in eps]).tobytes()).hexdigest()[:16]


def config1():
    cfg = configs.config(1)
    L = lattice.snap(cfg.a_raw, cfg.n)
    eps = E.sample(cfg.shape, cfg.n, L.a, L.delta, L.a_canon)
    kap = lattice.kvec_reduce(L, cfg.kpoints[0])
    t = time.time()
    _, nz, nnull = curl.dense_gep(L, kap, eps)
    dt = time.time() - t
    return {
        "_source": "scripts/make_golden.py: oracle.curl.dense_gep (plain definition, P:L1642-1646) on BASELINE config 1",
        "config": cfg.name, "n": list(cfg.n), "kappa": list(kap), "eps_sha256_16": eps_hash(eps),
        "null_count": nnull, "lambda": [float(x) for x in np.sort(nz)[:24]], "seconds": dt,
    }


def small_cases():
    """Dense A_r spectra at small grids of every config lattice (k-subsets)."""
    out = []
    for idx, n, kset in ((2, (8, 8, 8), [0, 4, 20]), (3, (8, 8, 6), [0, 6, 11]), (4, (8, 6, 6), [0, 12, 23])):
        cfg = configs.config(idx)
        L = lattice.snap(cfg.a_raw, n)
        eps = E.sample(cfg.shape, n, L.a, L.delta, L.a_canon)
        for ki in kset:
            if cfg.kappa_direct is not None:
                kap = lattice.kappa_from_raw(L, cfg.kappa_direct[ki])
            else:
                kap = lattice.kvec_reduce(L, cfg.kpoints[ki])
            Ar = spectral.Ar_dense(L, kap, eps)
            w = np.linalg.eigvalsh(Ar)
            if spectral.gamma_mode(L, kap) is not None:
                w = w[2:]
            out.append({"config": idx, "n": list(n), "k_index": ki, "kappa": list(kap),
                        "eps_sha256_16": eps_hash(eps), "lambda": [float(x) for x in w[:cfg.nev + 4]]})
    return {"_source": "scripts/make_golden.py: oracle.spectral.Ar_dense + eigvalsh (NFSEP, P:L2248-2251)",
            "cases": out}


if __name__ == "__main__":
    g = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(g, "small_nfsep_oracle.json"), "w") as f:
        json.dump(small_cases(), f, indent=1)
    with open(os.path.join(g, "config1_dense_oracle.json"), "w") as f:
        json.dump(config1(), f, indent=1)
