"""Solver-parameter sweep (block size, guard vectors) on a config: matvecs
and time per k-point, and agreement of the eigenvalues across settings.

    python scripts/sweep_solver.py --config 4 --kidx 5,12 --settings 1:2,2:2,2:4,4:2,4:4
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1806_10284_b200 as bnf  # noqa: E402
from bench import eps_for, kappas  # noqa: E402
from synthetic import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--kidx", default="5,12")
    ap.add_argument("--settings", default="1:2,2:2,2:4,4:2,4:4")
    ap.add_argument("--refine", type=int, default=1)
    ap.add_argument("--warm", type=int, default=0)
    args = ap.parse_args()
    cfg = configs.config(args.config)
    lat = bnf.Lattice(cfg.a_raw, cfg.n)
    eps = eps_for(cfg, lat)
    ks = kappas(cfg, lat)
    ref = {}
    for st in args.settings.split(","):
        b, g = (int(x) for x in st.split(":"))
        S = bnf.Solver(lat, block=b, guard=g, refine=args.refine, warm=args.warm)
        S.set_epsilon(eps)
        for ki in (int(x) for x in args.kidx.split(",")):
            torch.cuda.synchronize()
            t = time.perf_counter()
            lam, s = S.solve(ks[ki], cfg.nev, allow_noconv=True)
            dt = time.perf_counter() - t
            if ki not in ref:
                ref[ki] = lam
            dev = float(np.max(np.abs(lam - ref[ki]) / ref[ki]))
            print(json.dumps({"block": b, "guard": g, "k": ki, "sec": round(dt, 3), "matvecs": s["matvecs"],
                              "steps": s["outer_steps"], "inner": s["inner_iters"], "conv": s["converged"],
                              "res": s["max_residual"], "dev_vs_first": dev, "lam0": lam[0], "lamN": lam[-1]}),
                  flush=True)
        S.close()


if __name__ == "__main__":
    main()
