"""Micro-benchmark of the A_r apply (the hot operator) alone: per-pass CUDA
event times and algorithmic GB/s for each config grid.

    python scripts/bench_apply.py [--configs 1,2,3,4,5] [--b 1,4] [--reps 20]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1806_10284_b200 as bnf  # noqa: E402
from bench import PASS_BYTES, eps_for, kappas, load_peaks  # noqa: E402
from synthetic import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,4,5")
    ap.add_argument("--b", default="1,4")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    peak, _ = load_peaks()
    out = []
    for idx in [int(x) for x in args.configs.split(",")]:
        cfg = configs.config(idx)
        lat = bnf.Lattice(cfg.a_raw, cfg.n)
        n = lat.nn
        st = torch.cuda.Stream()
        S = bnf.Solver(lat, stream=st.cuda_stream, profile=1)
        S.set_epsilon(eps_for(cfg, lat))
        S.set_kappa(kappas(cfg, lat)[min(1, len(cfg.kpoints) - 1)])
        for b in [int(x) for x in args.b.split(",")]:
            y = torch.randn(b * 2 * n, dtype=torch.complex128, device="cuda")
            o = torch.empty_like(y)
            for _ in range(3):
                S.apply_Ar(y, o, b)
            S.kernel_times(reset=True)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(args.reps):
                S.apply_Ar(y, o, b)
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.reps
            kt = S.kernel_times(reset=True)
            per = {}
            for k, (kms, cnt) in kt.items():
                t = kms / cnt
                by = PASS_BYTES[k](n) * b if k in PASS_BYTES else 0
                per[k] = {"us": round(1000 * t, 1), "GBps": round(by / (t / 1e3) / 1e9, 1) if by else None}
            tot_bytes = sum(PASS_BYTES[k](n) for k in kt if k in PASS_BYTES) * b
            rec = {"config": cfg.name, "n": n, "b": b, "ms_per_apply": ms, "matvecs_per_s": b / (ms / 1e3),
                   "algorithmic_GBps": tot_bytes / (ms / 1e3) / 1e9, "frac_of_peak": tot_bytes / (ms / 1e3) / 1e9 / peak,
                   "passes": per}
            print(json.dumps(rec), flush=True)
            out.append(rec)
        S.close()


if __name__ == "__main__":
    main()
