"""The paper's grid-size table (PAPER.md, Table "Average time for
solving a GEP ... with various n1"): seconds per GEP (10 smallest eigenvalues,
tol 1e-12 / 1e-13) for n1 = n2 = n3 = 30, 36, ..., 120 on one B200, beside the
paper's K20c GPU column (context only: other hardware, other crystal -- the
paper does not say which).  Grids whose axis length has no register-FFT plan
run the generic Stockham passes (prime factors <= 31), e.g. 114 = 2 3 19.

    python scripts/grid_sweep.py [--sizes 30,36,...] [--shape fcc_diamond]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1806_10284_b200 as bnf  # noqa: E402
from synthetic import configs, eps as E  # noqa: E402

PAPER_K20C_S = {30: 4, 36: 5, 42: 6, 48: 8, 54: 10, 60: 13, 66: 15, 72: 19, 78: 26, 84: 28, 90: 32, 96: 39, 102: 48,
                108: 52, 114: 94, 120: 70}   # P:L2429-2438, K20c (context only)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default=",".join(str(k) for k in sorted(PAPER_K20C_S)))
    ap.add_argument("--shape", default="fcc_diamond")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = configs.config(2)
    K = cfg.kpoints[1]          # an X-U interior point (no degeneracy, no Gamma)
    res = []
    for nn in [int(x) for x in a.sizes.split(",")]:
        n = (nn, nn, nn)
        lat = bnf.Lattice(cfg.a_raw, n)
        eps = E.stacked(E.sample(a.shape, n, lat.a, lat.delta, lat.a_canon))
        S = bnf.Solver(lat)
        S.set_epsilon(eps)
        kap = lat.kvec_reduce(K)
        S.solve(kap, 10)                          # first call: autotune + graph capture
        t0 = time.perf_counter()
        lam, st = S.solve(kap, 10)
        dt = time.perf_counter() - t0
        line = {"n": nn, "seconds_per_gep": round(dt, 4), "paper_k20c_s": PAPER_K20C_S.get(nn),
                "matvecs": st["matvecs"], "converged": st["converged"], "max_residual": st["max_residual"],
                "lambda1": lam[0]}
        print(json.dumps(line), flush=True)
        res.append(line)
        S.close()
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
