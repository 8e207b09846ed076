"""Full band paths of the BASELINE configs through the k-path scheduler
(kpath.solve_path): wall time and k-points/s per config, eigenvalue
agreement with the oracle goldens where they exist (tests/golden/full_c*),
and the a-posteriori residual of every k-point.

    python scripts/path_bench.py [--configs 1,2,3,4,5] [--out profiles/r01_paths.json]
"""
import argparse
import glob
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1806_10284_b200 as bnf  # noqa: E402
from paper_1806_10284_b200 import kpath  # noqa: E402
from bench import eps_for, kappas  # noqa: E402
from synthetic import configs  # noqa: E402


def goldens():
    out = {}
    for f in glob.glob(os.path.join(ROOT, "tests", "golden", "full_c*_oracle.json")):
        with open(f) as fh:
            g = json.load(fh)
        out[(g["config"], tuple(round(x, 12) for x in g["kappa"]))] = g["lambda"]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--out", default=None)
    ap.add_argument("--warm", type=int, default=1)
    ap.add_argument("--per-gpu", default="1", help="concurrent solvers (streams) per GPU, or auto")
    ap.add_argument("--relax-inner", type=int, default=0)
    ap.add_argument("--method", type=int, default=0, help="0 inverse Lanczos (paper), 1 LOBPCG (NEXT-1)")
    ap.add_argument("--kmax", type=int, default=0, help="only the first kmax k-points of each path")
    ap.add_argument("--guard", type=int, default=None)
    ap.add_argument("--block", type=int, default=None)
    a = ap.parse_args()
    gold = goldens()
    res = []
    for idx in [int(x) for x in a.configs.split(",")]:
        cfg = configs.config(idx)
        lat = bnf.Lattice(cfg.a_raw, cfg.n)
        eps = eps_for(cfg, lat)
        ks = kappas(cfg, lat)
        if a.kmax:
            ks = ks[:a.kmax]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        extra = {"guard": a.guard} if a.guard is not None else {}
        if a.block is not None:
            extra["block"] = a.block
        pg = kpath.auto_per_gpu(cfg.n) if a.per_gpu == "auto" else int(a.per_gpu)
        recs = kpath.solve_path(cfg.a_raw, cfg.n, eps, ks, cfg.nev, device=0, warm=a.warm, per_gpu=pg,
                                relax_inner=a.relax_inner, method=a.method, **extra)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        failed = [(r.index, r.stats.get("error")) for r in recs if r.status == "failed"]
        for f in failed:
            print("FAILED k %d: %s" % f, flush=True)
        recs = [r for r in recs if r.status != "failed"] or recs
        dev = []
        for r in recs:
            key = (idx, tuple(round(x, 12) for x in r.kappa))
            if key in gold:
                g = np.asarray(gold[key][:len(r.lam)])
                dev.append(float(np.max(np.abs(np.asarray(r.lam[:len(g)]) - g) / g)))
        line = {"config": cfg.name, "grid": list(cfg.n), "nev": cfg.nev, "kpoints": len(ks), "seconds": round(dt, 3),
                "per_gpu": pg, "block": extra.get("block"), "guard": extra.get("guard"), "relax_inner": a.relax_inner, "method": a.method,
                "kpoints_per_s": len(ks) / dt, "status": sorted({r.status for r in recs}),
                "failed_kpoints": failed,
                "matvecs_per_kpoint": float(np.mean([r.stats.get("matvecs", 0) for r in recs])),
                "active_matvecs_per_kpoint": float(np.mean([r.stats.get("active_matvecs", 0) for r in recs])),
                "max_residual": max(r.stats.get("max_residual", float("nan")) for r in recs),
                "residual_per_k": [float("%.3g" % r.stats.get("max_residual", float("nan"))) for r in recs],
                "polish_steps_per_k": [int(r.stats.get("polish_steps", 0)) for r in recs],
                "golden_kpoints": len(dev), "max_rel_dev_vs_oracle": max(dev) if dev else None,
                "lambda_first_k": recs[0].lam[:4], "omega_over_2pi_first_k": kpath.frequencies(recs[0].lam[:4])}
        print(json.dumps(line), flush=True)
        res.append(line)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
