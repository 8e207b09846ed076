"""Benchmark of the hot path.

One *step* = one complete k-point solve (a0 per-k setup, a1-a5 A_r/M
applies inside a6 CG inside a7 block inverse Lanczos, a8 Rayleigh-Ritz +
residuals) of BASELINE config 4 (triclinic 128^3, seed-42 noise eps,
nev = 16) at the next k-point of its 24-point Gamma->(1/2,1/2,1/2) path.
Ranks take k-points round-robin (weak scaling, no data-path collective).

value  = matvecs/s (all ranks' A_r/M single-vector applications / max-rank
         device time); kpoints_per_s alongside.
e2e    = same metric through the C ABI with HOST buffers: eps uploaded
         (bnf_set_epsilon, host) and lambda read back every step.
roofline = the dominant kernel: algorithmic bytes / its CUDA-event time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synthetic import configs, eps as E  # noqa: E402

METRIC = "nullspace-free matvecs/s and k-points/s at 128^3 complex128; HBM GB/s vs peak"

# Algorithmic bytes per single-vector application, per pass (n = grid points).
# Reads + writes of complex128 (16 B) arrays; eps^{-1} is read as a uint8 index
# into a <=256-entry LUT (all BASELINE eps fields have 2 distinct values).
PASS_BYTES = {
    "zfwd": lambda n: 2 * 16 * n + 3 * 16 * n,       # read y1,y2; write 3 components
    "yfwd": lambda n: 2 * 3 * 16 * n,                 # in place, 3 components
    "xpass": lambda n: 2 * 3 * 16 * n + 3 * 1 * n,    # in place + eps^{-1} as uint8 LUT index
    "yadj": lambda n: 2 * 3 * 16 * n,
    "zadj": lambda n: 3 * 16 * n + 2 * 16 * n,        # read 3 components; write z1,z2
    # CG-fused variants (one CG iteration = zfwd_cg, yfwd, xpass_cg, yadj, zadj_cg)
    "zfwd_cg": lambda n: 4 * 16 * n + 2 * 16 * n + 3 * 16 * n,   # read r,p; write p; write 3 components
    "xpass_cg": lambda n: 2 * 3 * 16 * n + 3 * 1 * n,
    "zadj_cg": lambda n: 3 * 16 * n + 2 * 16 * n + 8 * 16 * n,   # read U, p; read+write x, r
    # fused y/x/y plane pass (plane.cu): one read + write of U, eps as uint8
    "plane": lambda n: 2 * 3 * 16 * n + 3 * 1 * n,
    "plane_cg": lambda n: 2 * 3 * 16 * n + 3 * 1 * n,
    "plane_l2": lambda n: 2 * 3 * 16 * n + 3 * 1 * n,     # same bytes, strips exchanged through L2
    "plane_l2_cg": lambda n: 2 * 3 * 16 * n + 3 * 1 * n,
    "plane_l2s": lambda n: 2 * 3 * 16 * n + 3 * 1 * n,    # L2 plane on a 2-CTA cluster per plane
    "plane_l2s_cg": lambda n: 2 * 3 * 16 * n + 3 * 1 * n,
    # warp-local FFT exchange variants of the L2 plane pass (smem / shuffles): same bytes
    "plane_w": lambda n: 2 * 3 * 16 * n + 3 * 1 * n,
    "plane_w_cg": lambda n: 2 * 3 * 16 * n + 3 * 1 * n,
    "plane_ws": lambda n: 2 * 3 * 16 * n + 3 * 1 * n,
    "plane_ws_cg": lambda n: 2 * 3 * 16 * n + 3 * 1 * n,
    "plane_t": lambda n: 2 * 3 * 16 * n + 3 * 1 * n,      # TMA-staged L2 plane pass (plane_tma.cu)
    "plane_t_cg": lambda n: 2 * 3 * 16 * n + 3 * 1 * n,
    "plane_ts": lambda n: 2 * 3 * 16 * n + 3 * 1 * n,     # TMA-staged, shuffle FFT exchange
    "plane_ts_cg": lambda n: 2 * 3 * 16 * n + 3 * 1 * n,
    "plane_tp": lambda n: 2 * 3 * 16 * n + 3 * 1 * n,      # TMA-staged, shuffles, two planes per CTA
    "plane_tp_cg": lambda n: 2 * 3 * 16 * n + 3 * 1 * n,
    # persistent pipelined z passes (zpass.cu); CG x update deferred into zfwd2_cg
    "zfwd2": lambda n: 2 * 16 * n + 3 * 16 * n,
    "zadj2": lambda n: 3 * 16 * n + 2 * 16 * n,
    "zfwd2_cg": lambda n: 6 * 16 * n + 4 * 16 * n + 3 * 16 * n,   # read r,p,x; write p,x; write U
    "zadj2_cg": lambda n: 3 * 16 * n + 4 * 16 * n,                 # read U, r; write r
    # persistent TMA-pipelined adjoint z pass (zpipe.cu): same bytes as zadj2
    "zadj3": lambda n: 3 * 16 * n + 2 * 16 * n,
    "zadj3_cg": lambda n: 3 * 16 * n + 4 * 16 * n,
}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def workload(idx):
    cfg = configs.config(idx)
    return cfg


def kappas(cfg, lat):
    if cfg.kappa_direct is not None:
        return [lat.kappa_from_raw(k) for k in cfg.kappa_direct]
    return [lat.kvec_reduce(K) for K in cfg.kpoints]


def eps_for(cfg, lat):
    return E.stacked(E.sample(cfg.shape, cfg.n, lat.a, lat.delta, lat.a_canon))


# ----------------------------------------------------------------- oracle arm
def host_info():
    """CPU model, core count and library versions of the host the oracle runs on."""
    import platform

    import scipy
    model = platform.processor() or "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu": model, "nproc": os.cpu_count(), "numpy": np.__version__, "scipy": scipy.__version__,
            "fft": "scipy.fft (pocketfft)", "python": platform.python_version()}


def oracle_rate(cfg, seconds=15.0, max_matvecs=30, min_matvecs=2, threads=1, workers=1):
    """Oracle (numpy/scipy, as it stands) matvecs/s on a bounded sample of
    the same workload: A_r applications at the first k-point.  threads /
    workers: the oracle's execution knobs (oracle/fftop.py ORACLE_THREADS,
    ORACLE_FFT_WORKERS; bit-identical results).  Returns (rate, count, wall
    seconds, effective cores = process CPU time / wall)."""
    from oracle import fftop, lattice as olat
    O = olat.snap(cfg.a_raw, cfg.n)
    eps = E.sample(cfg.shape, cfg.n, O.a, O.delta, O.a_canon)
    if cfg.kappa_direct is not None:
        kap = olat.kappa_from_raw(O, cfg.kappa_direct[1])
    else:
        kap = olat.kvec_reduce(O, cfg.kpoints[0])
    op = fftop.NFSEPOperator(O, kap, eps)
    y = np.random.default_rng(0).standard_normal(2 * O.nn) + 0j
    keep = (fftop._THREADS, fftop._WORKERS)
    fftop._THREADS, fftop._WORKERS = threads, workers
    try:
        t0 = time.perf_counter()
        c0 = time.process_time()
        cnt = 0
        while cnt < max_matvecs and (cnt < min_matvecs or time.perf_counter() - t0 < seconds):
            y = op.Ar(y)
            y /= np.linalg.norm(y)
            cnt += 1
        dt = time.perf_counter() - t0
        cores = (time.process_time() - c0) / dt
    finally:
        fftop._THREADS, fftop._WORKERS = keep
    return cnt / dt, cnt, dt, cores


def cpu_baseline_pair(cfg, seconds=12.0):
    """The oracle single-threaded and on all host cores (3 component threads x
    nproc/3 FFT workers), SURVEY §8(d).  Reported as a baseline, not a target."""
    nproc = os.cpu_count() or 1
    r1, c1, d1, co1 = oracle_rate(cfg, seconds=seconds, max_matvecs=20)
    ra, ca, da, coa = oracle_rate(cfg, seconds=seconds, max_matvecs=40, threads=3, workers=max(1, nproc // 3))
    return {"value": ra, "unit": "matvecs/s", "cores": round(coa, 2), "kind": "oracle",
            "sample": "%d oracle A_r applications at %s, k-point 1 (scipy.fft, 3 component threads x %d FFT "
                      "workers, %.1f s)" % (ca, cfg.name, max(1, nproc // 3), da),
            "single_thread": {"value": r1, "cores": round(co1, 2), "applications": c1, "seconds": round(d1, 2)},
            "host": host_info(), "note": "baseline, not a target (plain fp64 NumPy/SciPy oracle)"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg = workload(args.config)
    total = 0
    tt = 0.0
    cores = []
    for _ in range(args.warmup):
        oracle_rate(cfg, seconds=1.0, max_matvecs=2, min_matvecs=1)
    for _ in range(args.steps):
        r, c, dt, co = oracle_rate(cfg, seconds=3.0, max_matvecs=6, min_matvecs=2)
        total += c
        tt += dt
        cores.append(co)
    v = total / tt
    sample = "%d oracle A_r applications (scipy.fft, 1 thread) at %s, %d steps of <= 6" % (total, cfg.name,
                                                                                           args.steps)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "matvecs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic", "config": {"workload": cfg.name, "grid": list(cfg.n)},
        "cpu_baseline": {"value": v, "unit": "matvecs/s", "cores": round(max(cores), 2), "kind": "oracle",
                         "sample": sample, "host": host_info()},
        "e2e": {"value": v, "unit": "matvecs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours")
    # defaults from profiles/r03_bench_block_sweep.jsonl (128^3, k12-k15): block 1 needs 22 % fewer
    # operator applications per k-point than block 2 (2766 vs 3570) at 5 % lower matvec rate; two
    # concurrent solvers per GPU recover most of that rate (the b = 1 launches underfill the GPU)
    ap.add_argument("--block", type=int, default=1)
    ap.add_argument("--guard", type=int, default=2)
    ap.add_argument("--per-gpu", type=int, default=2,
                    help="concurrent solvers (one stream + host thread each) per GPU; a step solves one k-point each")
    ap.add_argument("--warm", type=int, default=1,
                    help="start each k-point from the previous one's Ritz vectors (DESIGN R17)")
    ap.add_argument("--kstart", type=int, default=12, help="path index of the first timed k-point")
    ap.add_argument("--relax-inner", type=int, default=0,
                    help="NEXT-1 inexact inner CG (bnf_opts.relax_inner); default 0 = the paper's fixed 1e-13")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch this command under torchrun (rank 0 prints the line)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.run(cmd).returncode)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%d (launch one process per GPU)" % (args.gpus, world))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_1806_10284_b200 as bnf
    from paper_1806_10284_b200 import kpath

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = workload(args.config)
    lat = bnf.Lattice(cfg.a_raw, cfg.n)
    eps = eps_for(cfg, lat)
    ks = kappas(cfg, lat)
    C = max(1, args.per_gpu)
    streams = [torch.cuda.Stream() for _ in range(C)]
    solvers = []
    for c in range(C):
        Sc = bnf.Solver(lat, device=local, stream=streams[c].cuda_stream, profile=0, block=args.block,
                        guard=args.guard, warm=args.warm, relax_inner=args.relax_inner)
        Sc.set_epsilon(eps)
        solvers.append(Sc)
    S, stream = solvers[0], streams[0]
    nev = cfg.nev

    share = kpath.assign(ks, world)[rank]   # LPT share of the path (no data-path collective)

    # the timed steps start at path point --kstart (k12 by default: the middle of the path, whose oracle
    # golden exists; with --steps 12 or more the timed k-points also cover k23 and k0 = Gamma).  With C
    # solvers per GPU, solver c walks its own contiguous run of the share (warm starts stay adjacent):
    # its timed k-points start C * steps positions after solver c - 1's.
    off = (share.index(args.kstart) - args.warmup) % len(share) if args.kstart in share else 0

    def kidx(step, c=0):
        return share[(step + c * args.steps + off) % len(share)]

    def barrier():
        if world > 1:
            dist.barrier()

    def run_all(fn):
        """fn(c) on every solver, concurrently (one host thread each; the C ABI releases the GIL)."""
        if C == 1:
            return [fn(0)]
        out = [None] * C
        err = []

        def th(c):
            try:
                out[c] = fn(c)
            except BaseException as e:   # re-raised below
                err.append(e)
        ths = [threading.Thread(target=th, args=(c,)) for c in range(C)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        if err:
            raise err[0]
        return out

    # warm-up (untimed)
    run_all(lambda c: [solvers[c].solve(ks[kidx(s_, c)], nev, allow_noconv=True) for s_ in range(args.warmup)])
    for Sc in solvers:
        Sc.kernel_times(reset=True)
    # timed: device-resident inputs
    barrier()
    torch.cuda.synchronize()
    main = torch.cuda.current_stream()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)

    def timed(c):
        res = []
        for s_ in range(args.steps):
            k = kidx(args.warmup + s_, c)
            lam, st = solvers[c].solve(ks[k], nev, allow_noconv=True)
            res.append((k, lam, st))
        return res
    with ClockSampler(local) as clk:
        ev0.record(main)
        for st_ in streams:
            st_.wait_event(ev0)
        per = run_all(timed)
        for st_ in streams:
            main.wait_stream(st_)
        ev1.record(main)
        torch.cuda.synchronize()
    barrier()
    ms = ev0.elapsed_time(ev1)
    mv = sum(st["matvecs"] for r in per for _, _, st in r)
    launches = sum(st["kernel_launches"] for r in per for _, _, st in r)
    stats = [st for r in per for _, _, st in r]
    lams = [(k, lam) for r in per for k, lam, _ in r]
    # Kernel profile (roofline): one more k-point of this rank's share, run by solver 0 alone with
    # per-kernel CUDA events on its stream.  The timed steps above run the CG loop as a CUDA graph
    # (no per-iteration host round trip); this pass launches the same kernels eagerly so each one can
    # be bracketed by events.
    S.set_profile(1)
    S.kernel_times(reset=True)
    evp0 = torch.cuda.Event(enable_timing=True)
    evp1 = torch.cuda.Event(enable_timing=True)
    evp0.record(stream)
    _, stp = S.solve(ks[kidx(args.warmup + args.steps)], nev, allow_noconv=True)
    evp1.record(stream)
    torch.cuda.synchronize()
    ms_prof = evp0.elapsed_time(evp1)
    ktimes = S.kernel_times(reset=True)
    S.set_profile(0)
    mv_prof = stp["matvecs"]
    t_all = torch.tensor([ms, mv, args.steps], dtype=torch.float64, device="cuda")
    if world > 1:
        tmax = t_all.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t_all.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        ms_max = float(tmax[0])
        mv_tot = float(tsum[1])
    else:
        ms_max, mv_tot = ms, float(mv)
    value = mv_tot / (ms_max / 1000.0)
    kps = world * C * args.steps / (ms_max / 1000.0)

    # e2e: host buffers through the C ABI (eps H2D + lambda D2H inside the timed region)
    e2e = None
    if not args.no_e2e:
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()

        def e2e_run(c):
            m = 0
            for s_ in range(args.steps):
                solvers[c].set_epsilon(eps)      # host -> device every step
                lam, st = solvers[c].solve(ks[kidx(args.warmup + s_, c)], nev, allow_noconv=True)   # lambda -> host
                m += st["matvecs"]
            return m
        mv2 = sum(run_all(e2e_run))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        t2 = torch.tensor([dt, mv2], dtype=torch.float64, device="cuda")
        if world > 1:
            m2 = t2.clone()
            dist.all_reduce(m2, op=dist.ReduceOp.MAX)
            s2 = t2.clone()
            dist.all_reduce(s2, op=dist.ReduceOp.SUM)
            dt, mv2 = float(m2[0]), float(s2[1])
        e2e = {"value": mv2 / dt, "unit": "matvecs/s", "h2d_bytes_per_step": int(eps.nbytes) * C,
               "d2h_bytes_per_step": int(8 * nev * C), "kpoints_per_s": world * C * args.steps / dt}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # roofline of the dominant kernel
    peak, peak_src = load_peaks()
    n = lat.nn
    dom = max(ktimes.items(), key=lambda kv: kv[1][0]) if ktimes else None
    # vectors served by the CG-fused passes vs the plain ones (plain y/x passes serve both)
    zc = sum(v[1] for k, v in ktimes.items() if k.startswith("zfwd") and k.endswith("_cg"))
    zp = sum(v[1] for k, v in ktimes.items() if k.startswith("zfwd") and not k.endswith("_cg"))
    mv_cg = mv_prof * zc / (zc + zp) if zc + zp > 0 else 0
    def vecs(k):   # vectors served by pass k ("_cg" variants serve CG iterations only)
        if k.endswith("_cg"):
            return mv_cg
        if k + "_cg" in PASS_BYTES:
            return mv_prof - mv_cg
        return mv_prof
    roof = None
    if dom and dom[0] in PASS_BYTES:
        name, (kms, kcnt) = dom
        per_vec = PASS_BYTES[name](n)
        # every apply launches each pass once per batch: the pass's vector count is
        # the matvecs it served (fused-CG and plain variants are timed separately)
        total_bytes = per_vec * vecs(name)
        achieved = total_bytes / (kms / 1000.0) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                tj = json.load(f)
            if tj.get(name) is not None:
                # DRAM bytes per launch from the ncu capture, scaled to this launch's vector count
                vcap = float(tj.get("_vectors_per_launch", 2))
                traffic = tj[name] * (total_bytes / kcnt) / (per_vec * vcap)
        roof = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "bytes_per_launch": total_bytes / kcnt,
                "avg_launch_us": 1000.0 * kms / kcnt, "peak_source": peak_src,
                "share_of_step": kms / ms_prof,
                "timing": "per-kernel CUDA events over one profiled k-point solve (eager launches)"}
    matvec_ms = sum(v[0] for k, v in ktimes.items() if k in PASS_BYTES)
    matvec_bytes = sum(PASS_BYTES[k](n) * vecs(k) for k in ktimes if k in PASS_BYTES)
    cpu = None
    if not args.no_cpu and world == 1:   # the oracle baseline is timed at N = 1 only
        cpu = cpu_baseline_pair(cfg)
    # timed k-points with an oracle golden (scripts/make_golden_full.py): eigenvalue deviation
    devs = []
    for ki, lam in lams:
        gp = os.path.join(ROOT, "tests", "golden", "full_c%d_k%d_oracle.json" % (args.config, ki))
        if os.path.exists(gp):
            with open(gp) as f:
                g = json.load(f)
            gl = np.asarray(g["lambda"][:nev])
            devs.append(float(np.max(np.abs(np.asarray(lam[:len(gl)]) - gl) / gl)))
    golden = {"timed_kpoints_with_golden": len(devs), "timed_kpoints": len(lams),
              "max_rel_dev_vs_oracle": max(devs) if devs else None}
    line = {
        "metric": METRIC, "value": value, "unit": "matvecs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "kpoints_per_step": C, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": cfg.name, "grid": list(cfg.n), "nev": nev, "kpoints_on_path": len(ks),
                   "block": args.block, "guard": args.guard, "tol_outer": 1e-12, "tol_inner": 1e-13,
                   "warm_start": bool(args.warm), "relax_inner": bool(args.relax_inner),
                   "l2": "inputs larger than L2 (Krylov basis and work arrays >> 126 MB)",
                   "solvers_per_gpu": C,
                   "parallelism": "k-point replicas x%d (x%d concurrent solvers per GPU)" % (world, C)},
        "kpoints_per_s": kps,
        "matvec_pipeline": {"ms_total": matvec_ms, "algorithmic_GBps": matvec_bytes / (matvec_ms / 1e3) / 1e9
                            if matvec_ms else None, "share_of_step": matvec_ms / ms_prof,
                            "profiled_step_ms": ms_prof, "profiled_matvecs": mv_prof},
        "roofline": roof,
        "golden_check": golden,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "solver": {"matvecs_per_kpoint": mv / (C * args.steps),
                   "outer_steps": [s_["outer_steps"] for s_ in stats],
                   "converged": all(s_["converged"] for s_ in stats),
                   "max_residual": max(s_["max_residual"] for s_ in stats)},
        "kernel_ms": {k: round(v[0], 3) for k, v in ktimes.items()},
        "middle": ("plane_l2s" if "plane_l2s_cg" in ktimes else "plane_tp" if "plane_tp_cg" in ktimes else "plane_ts" if "plane_ts_cg" in ktimes else "plane_t" if "plane_t_cg" in ktimes else "plane_ws" if "plane_ws_cg" in ktimes else "plane_w" if "plane_w_cg" in ktimes
                   else "plane_l2" if "plane_l2_cg" in ktimes else "plane_cluster" if "plane_cg" in ktimes
                   else "y/x/y"),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
