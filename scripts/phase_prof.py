"""Per-phase cycle breakdown of the plane pass (diagnostics).

    BNF_PHASE_PROF=1 python scripts/phase_prof.py [--config 4] [--b 2] [--reps 5]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("BNF_PHASE_PROF", "1")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1806_10284_b200 as bnf  # noqa: E402
from bench import eps_for, kappas  # noqa: E402
from synthetic import configs  # noqa: E402

NAMES = ["load+yFFT", "twiddle", "barrier1", "dsmem Y->X", "barrier2", "xFFT", "eps", "xFFT*", "barrier3",
         "dsmem X->Y", "barrier4", "tw*+yFFT*", "stores"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--b", type=int, default=2)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    cfg = configs.config(a.config)
    lat = bnf.Lattice(cfg.a_raw, cfg.n)
    S = bnf.Solver(lat)
    S.set_epsilon(eps_for(cfg, lat))
    ks = kappas(cfg, lat)
    S.set_kappa(ks[min(1, len(ks) - 1)])
    n = lat.nn
    y = torch.randn(a.b * 2 * n, dtype=torch.complex128, device="cuda")
    o = torch.empty_like(y)
    S.apply_Ar(y, o, a.b)
    S.phase_counters()
    for _ in range(a.reps):
        S.apply_Ar(y, o, a.b)
    c = S.phase_counters().astype(np.float64)
    ctas = c[15]
    tot = c[:13].sum()
    print("config %s b=%d: %d CTAs, %.0f cycles per CTA" % (cfg.name, a.b, ctas, tot / ctas))
    for k, nm in enumerate(NAMES):
        print("  %-12s %8.0f cyc/CTA  %5.1f%%" % (nm, c[k] / ctas, 100 * c[k] / tot))


if __name__ == "__main__":
    main()
