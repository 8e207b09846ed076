"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
one A_r and M apply on the fast path at 64^3 (z passes + cluster plane pass),
one CG-fused solve at 12^3 and at 64^3 (graph CG loop, fused reductions).

    compute-sanitizer --tool memcheck python scripts/sanitize_case.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1806_10284_b200 as bnf  # noqa: E402
from bench import eps_for, kappas  # noqa: E402
from synthetic import configs  # noqa: E402


def main():
    quick = "--quick" in sys.argv
    for idx, nev in ((1, 4), (2, 2)):
        cfg = configs.config(idx)
        lat = bnf.Lattice(cfg.a_raw, cfg.n)
        S = bnf.Solver(lat, block=2, guard=0, max_outer=3 if quick else 60)
        S.set_epsilon(eps_for(cfg, lat))
        kap = kappas(cfg, lat)[0]
        S.set_kappa(kap)
        n = lat.nn
        y = torch.randn(2 * 2 * n, dtype=torch.complex128, device="cuda")
        o = torch.empty_like(y)
        S.apply_Ar(y, o, 2, bnf.OP_AR)
        S.apply_Ar(y, o, 2, bnf.OP_M)
        lam, st = S.solve(kap, nev, allow_noconv=True)
        torch.cuda.synchronize()
        print(cfg.name, "ok", lam[:2], st["matvecs"], flush=True)
        S.close()


if __name__ == "__main__":
    main()
