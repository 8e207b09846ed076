"""NEXT-2 second workload: the gyroid photonic crystal
on the BCC lattice, its band structure along Gamma-H-N-Gamma-P-H for a sweep
of the material permittivity (3 ... 30), and the complete band gaps of each
(kpath.band_gaps, omega / 2 pi units).  The paper shows the sweep as a
figure only (no numbers), so this reports, it does not compare.

    python scripts/eps_sweep.py [--n 32] [--nev 10] [--kpoints 30] [--eps 3,5,8,10,13,16,20,25,30]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1806_10284_b200 as bnf  # noqa: E402
from paper_1806_10284_b200 import kpath  # noqa: E402
from synthetic import configs, eps as E  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--nev", type=int, default=10)
    ap.add_argument("--eps", default="3,5,8,10,13,16,20,25,30")
    ap.add_argument("--per-gpu", type=int, default=1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = configs.config(3)                       # BCC vectors and the Gamma-H-N-Gamma-P-H path
    n = (a.n, a.n, a.n)
    lat = bnf.Lattice(cfg.a_raw, n)
    ks = [lat.kvec_reduce(K) for K in cfg.kpoints]
    res = []
    for e in [float(x) for x in a.eps.split(",")]:
        eps = E.stacked(E.sample("gyroid:%g" % e, n, lat.a, lat.delta, lat.a_canon))
        t0 = time.perf_counter()
        recs = kpath.solve_path(cfg.a_raw, n, eps, ks, a.nev, device=0, warm=1, per_gpu=a.per_gpu)
        dt = time.perf_counter() - t0
        gaps = kpath.band_gaps(recs)
        line = {"eps": e, "grid": list(n), "kpoints": len(ks), "seconds": round(dt, 3),
                "status": sorted({r.status for r in recs}),
                "max_residual": max(r.stats["max_residual"] for r in recs),
                "gaps": [{"between_bands": [g[0] + 1, g[0] + 2], "omega_lo": g[1], "omega_hi": g[2], "width": g[3],
                          "gap_to_midgap": g[4]} for g in gaps[:3]],
                "omega_max_band1": max(kpath.frequencies(r.lam)[0] for r in recs)}
        print(json.dumps(line), flush=True)
        res.append(line)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
