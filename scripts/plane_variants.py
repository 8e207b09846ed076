"""Real-space middle variants side by side (one config grid, block b): for
each forced variant, the per-kernel CUDA-event times of one CG-fused solve
step mix are not needed -- this times bnf_cg_solve (fused CG, eager, profile
on) for a fixed number of iterations and reports every pass's mean launch
time and algorithmic GB/s, plus the max deviation of x between variants.

    python scripts/plane_variants.py [--config 4] [--b 2] [--iters 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1806_10284_b200 as bnf  # noqa: E402
from bench import PASS_BYTES, eps_for, kappas, load_peaks  # noqa: E402
from synthetic import configs  # noqa: E402

VARIANTS = {"yxy": {"BNF_NO_PLANE": "1"}, "cluster": {"BNF_PLANE": "1"},
            "l2": {"BNF_PLANE": "1", "BNF_PLANE_L2": "1"}, "warp_smem": {"BNF_PLANE_W": "1"},
            "warp_shfl": {"BNF_PLANE_W": "2"}, "tma": {"BNF_PLANE_T": "1"}, "tma_shfl": {"BNF_PLANE_T": "2"},
            "tma_pair": {"BNF_PLANE_T": "3"},
           "l2_split": {"BNF_PLANE": "1", "BNF_PLANE_L2": "1", "BNF_PLANE_SPLIT": "2"},
           "l2_rs": {"BNF_PLANE": "1", "BNF_PLANE_L2": "1", "BNF_PLANE_RS": "1"},
           "l2_xeo": {"BNF_PLANE": "1", "BNF_PLANE_L2": "1", "BNF_PLANE_XEO": "1"},
           "l2_xeo_rs": {"BNF_PLANE": "1", "BNF_PLANE_L2": "1", "BNF_PLANE_XEO": "1", "BNF_PLANE_RS": "1"},
           "l2_ld1": {"BNF_PLANE": "1", "BNF_PLANE_L2": "1", "BNF_PLANE_LD": "1"},
           "l2_ld2": {"BNF_PLANE": "1", "BNF_PLANE_L2": "1", "BNF_PLANE_LD": "2"},
           "l2_ld3": {"BNF_PLANE": "1", "BNF_PLANE_L2": "1", "BNF_PLANE_LD": "3"},
           "l2_noxw": {"BNF_PLANE": "1", "BNF_PLANE_L2": "1", "BNF_PLANE_LD": "4"},
           "l2_noxw_ld2": {"BNF_PLANE": "1", "BNF_PLANE_L2": "1", "BNF_PLANE_LD": "6"},
           "l2_noxw_ld3": {"BNF_PLANE": "1", "BNF_PLANE_L2": "1", "BNF_PLANE_LD": "7"}}
# z-pass register-budget variants (BNF_ZCFG bits, kernels.cuh zcfg), with the L2 plane middle
for _z in (5, 1029, 517, 2053, 2049, 3077, 3073):
    VARIANTS["z%d" % _z] = {"BNF_PLANE": "1", "BNF_PLANE_L2": "1", "BNF_ZCFG": str(_z)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--b", type=int, default=2)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--variants", default=",".join(VARIANTS))
    args = ap.parse_args()
    peak, _ = load_peaks()
    cfg = configs.config(args.config)
    lat = bnf.Lattice(cfg.a_raw, cfg.n)
    n = lat.nn
    eps = eps_for(cfg, lat)
    kap = kappas(cfg, lat)[min(7, len(kappas(cfg, lat)) - 1)]
    g = torch.Generator(device="cuda").manual_seed(1)
    c = torch.randn(args.b * 2 * n, dtype=torch.complex128, device="cuda", generator=g)
    ref = None
    for name in args.variants.split(","):
        for k in ("BNF_PLANE", "BNF_PLANE_L2", "BNF_NO_PLANE", "BNF_PLANE_W", "BNF_PLANE_T", "BNF_PLANE_SPLIT",
                  "BNF_PLANE_RS", "BNF_PLANE_XEO", "BNF_PLANE_LD", "BNF_ZCFG"):
            os.environ.pop(k, None)
        os.environ.update(VARIANTS[name])
        st = torch.cuda.Stream()
        S = bnf.Solver(lat, stream=st.cuda_stream, profile=1)
        S.set_epsilon(eps)
        S.set_kappa(kap)
        x = torch.empty_like(c)
        S.cg_solve(c, x, args.b, 3)               # warm-up (and autotune bypass)
        S.kernel_times(reset=True)
        S.cg_solve(c, x, args.b, args.iters)
        torch.cuda.synchronize()
        kt = S.kernel_times(reset=True)
        dev = None
        if ref is None:
            ref = x.clone()
        else:
            dev = float((x - ref).abs().max() / ref.abs().max())
        per = {}
        tot = 0.0
        for k, (kms, cnt) in kt.items():
            t = kms / cnt
            by = PASS_BYTES[k](n) * args.b if k in PASS_BYTES else 0
            tot += kms
            per[k] = {"us": round(1000 * t, 1), "launches": cnt,
                      "frac": round(by / (t / 1e3) / 1e9 / peak, 3) if by else None}
        print(json.dumps({"variant": name, "config": cfg.name, "b": args.b, "iters": args.iters,
                          "ms_per_iter": tot / args.iters, "dev_vs_first": dev, "passes": per}), flush=True)
        S.close()
        for k in VARIANTS[name]:
            os.environ.pop(k, None)


if __name__ == "__main__":
    main()
