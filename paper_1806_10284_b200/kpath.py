"""k-path scheduler ("for each
wave vector ... partition each segment").

The k-points of a band path are independent generalized eigenproblems, so
the path is sharded across ranks (one process per GPU) with NO data-path
collective: each rank solves its own k-points through the C ABI
(``Solver.solve``) and only the per-k results (nev doubles + stats) are
gathered at the end.  This module holds only host logic:

* ``assign``      -- deterministic k -> rank assignment: longest-processing-
                     time-first over a per-k cost estimate (Gamma and other
                     high-symmetry points with degenerate / masked modes are
                     heavier), ties broken by k index;
* ``run_path``    -- drive a ``solve(kappa) -> (lam, stats)`` callable over
                     this rank's share, with per-k retry and a JSONL
                     checkpoint (resume skips finished k);
* ``StealQueue``  -- dynamic balancing on top of the LPT shares: every rank
                     walks its own share front to back through an atomic
                     per-rank cursor in the process group's key-value store,
                     and a rank whose share is exhausted takes the next
                     unclaimed k of the rank with the most work left (each k
                     is claimed exactly once; owners keep contiguous runs,
                     so warm starts stay local);
* ``gather``      -- merge every rank's records into path order
                     (torch.distributed object gather; gloo or nccl).
"""
from __future__ import annotations

import json
import math
import os
import time
from dataclasses import dataclass, field


def kpoint_cost(kappa, tol=1e-12):
    """Relative cost estimate of one k-point solve.  Points with every
    kappa_l integral (Gamma, R6: masked mode) or half-integral (zone
    boundary: exact degeneracies) need more Lanczos steps."""
    def frac(x):
        return abs(x - round(x))
    c = 1.0
    if all(frac(k) < tol for k in kappa):
        c += 0.5
    half = sum(1 for k in kappa if abs(frac(k) - 0.5) < tol)
    c += 0.15 * half
    return c


def assign(kappas, world, costs=None):
    """LPT assignment of k indices to ``world`` ranks.  Returns a list of
    index lists (one per rank), each in ascending k order.  Deterministic."""
    if world < 1:
        raise ValueError("world must be >= 1")
    costs = list(costs) if costs is not None else [kpoint_cost(k) for k in kappas]
    order = sorted(range(len(kappas)), key=lambda i: (-costs[i], i))
    load = [0.0] * world
    share = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda q: (load[q], q))
        share[r].append(i)
        load[r] += costs[i]
    return [sorted(s) for s in share]


class StealQueue:
    """Exactly-once k claiming with work stealing (see module docstring).
    ``store``: a torch.distributed Store (``add`` is atomic across ranks), or
    None for a single process.  ``shares``: the LPT shares (``assign``)."""

    def __init__(self, shares, rank, store=None, prefix="kpath"):
        self.shares = [list(s) for s in shares]
        self.rank = rank
        self.store = store
        self.prefix = prefix
        self._local = [0] * len(self.shares)

    def _add(self, r, inc):
        if self.store is None:
            v = self._local[r]
            self._local[r] += inc
            return v + inc
        return int(self.store.add("%s/cursor%d" % (self.prefix, r), inc))

    def _claim(self, r):
        pos = self._add(r, 1) - 1
        return self.shares[r][pos] if pos < len(self.shares[r]) else None

    def __iter__(self):
        while True:
            i = self._claim(self.rank)
            if i is not None:
                yield i
                continue
            # own share exhausted: help the rank with the most unclaimed k
            left = [(len(s) - self._add(r, 0), r) for r, s in enumerate(self.shares) if r != self.rank]
            left = [x for x in left if x[0] > 0]
            if not left:
                return
            _, victim = max(left)
            i = self._claim(victim)
            if i is not None:
                yield i


def run_meta(nev, eps=None, **opts):
    """Identity of a run for checkpoint reuse: nev, a hash of eps, options."""
    import hashlib
    h = hashlib.sha256()
    h.update(json.dumps({"nev": int(nev), **{k: opts[k] for k in sorted(opts)}}, default=str).encode())
    if eps is not None:
        import numpy as np
        h.update(np.ascontiguousarray(eps).tobytes())
    return h.hexdigest()[:16]


@dataclass
class KRecord:
    index: int
    kappa: tuple
    status: str                 # "ok" | "noconv" | "failed"
    lam: list = field(default_factory=list)
    stats: dict = field(default_factory=dict)
    rank: int = 0
    attempts: int = 1
    seconds: float = 0.0
    meta: str = ""              # run_meta() of the run that produced it

    def to_json(self):
        return json.dumps({"index": self.index, "kappa": list(self.kappa), "status": self.status,
                           "lam": list(self.lam), "stats": self.stats, "rank": self.rank,
                           "attempts": self.attempts, "seconds": self.seconds, "meta": self.meta})

    @staticmethod
    def from_json(line):
        d = json.loads(line)
        return KRecord(d["index"], tuple(d["kappa"]), d["status"], d["lam"], d["stats"], d["rank"],
                       d["attempts"], d["seconds"], d.get("meta", ""))


def load_checkpoint(paths, kappas=None, meta=None):
    """Finished records of previous runs (status ok or noconv), by k index.
    ``paths``: one JSONL path or a list (every rank's file, so a resume with
    another world size or stealing pattern still finds each finished k).  A
    record is reused only if its kappa equals ``kappas[index]`` and its
    ``meta`` equals ``meta`` (when given): a changed path, nev, eps or
    option set is never served from a stale checkpoint."""
    if isinstance(paths, str) or paths is None:
        paths = [paths]
    done = {}
    for path in paths:
        if not path or not os.path.exists(path):
            continue
        with open(path) as f:
            for line in f:
                line = line.strip()
                if not line:
                    continue
                try:
                    r = KRecord.from_json(line)
                except (ValueError, KeyError, TypeError):
                    continue   # torn last line of an interrupted run
                if r.status not in ("ok", "noconv"):
                    continue
                if meta is not None and r.meta != meta:
                    continue
                if kappas is not None and (r.index >= len(kappas) or
                                           tuple(float(x) for x in kappas[r.index]) != tuple(r.kappa)):
                    continue
                done[r.index] = r
    return done


def run_path(solve, kappas, indices, rank=0, checkpoint=None, retries=1, clock=time.perf_counter, meta="",
             resume_from=None):
    """Solve the k-points ``indices`` (this rank's share, or a StealQueue)
    with ``solve``.

    ``solve(kappa)`` returns ``(lam, stats_dict)``; ``stats_dict["rc"]`` may
    mark non-convergence (6 = BNF_ENOCONV).  An exception is retried
    ``retries`` times and then recorded as ``failed`` (the path continues).
    With ``checkpoint`` (a per-rank JSONL path) new records are appended as
    they complete, and k finished by a previous run with the same ``meta``
    and kappa (in ``checkpoint`` or any file of ``resume_from``) are skipped."""
    done = load_checkpoint(list(resume_from or []) + [checkpoint], kappas, meta)
    out = []
    fh = open(checkpoint, "a") if checkpoint else None
    try:
        for i in indices:
            if i in done:
                out.append(done[i])
                continue
            kap = tuple(float(x) for x in kappas[i])
            rec = None
            for attempt in range(1, retries + 2):
                t0 = clock()
                try:
                    lam, st = solve(kap)
                    status = "noconv" if st.get("rc", 0) == 6 else "ok"
                    rec = KRecord(i, kap, status, [float(x) for x in lam], dict(st), rank, attempt, clock() - t0,
                                  meta)
                    break
                except Exception as e:  # noqa: BLE001 -- recorded, path continues
                    rec = KRecord(i, kap, "failed", [], {"error": str(e)}, rank, attempt, clock() - t0, meta)
            out.append(rec)
            if fh:
                fh.write(rec.to_json() + "\n")
                fh.flush()
    finally:
        if fh:
            fh.close()
    return out


def merge(per_rank_records, nk):
    """Path-ordered list of length nk (None where a k was not solved)."""
    res = [None] * nk
    for recs in per_rank_records:
        for r in recs:
            if res[r.index] is None or (res[r.index].status != "ok" and r.status == "ok"):
                res[r.index] = r
    return res


def gather(records, nk, group=None):
    """Gather every rank's records (torch.distributed, any backend) and
    return the merged path on every rank.  Single process: just merge."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return merge([records], nk)
    world = dist.get_world_size(group)
    payload = [r.to_json() for r in records]
    allp = [None] * world
    dist.all_gather_object(allp, payload, group=group)
    return merge([[KRecord.from_json(x) for x in p] for p in allp], nk)


def band_gaps(records, nbands=None):
    """Complete band gaps of a path (NEXT-2): for each pair of
    consecutive bands (i, i+1), gap_i = min_k omega_{i+1}(k) - max_k omega_i(k)
    in omega / (2 pi) units.  Returns a list of (i, lower edge,
    upper edge, width, width / midgap) for the positive gaps, widest first."""
    om = [frequencies(r.lam if hasattr(r, "lam") else r) for r in records if r is not None]
    if not om:
        return []
    nb = min(len(o) for o in om) if nbands is None else nbands
    out = []
    for i in range(nb - 1):
        lo = max(o[i] for o in om)
        hi = min(o[i + 1] for o in om)
        if hi > lo:
            out.append((i, lo, hi, hi - lo, 2.0 * (hi - lo) / (hi + lo)))
    return sorted(out, key=lambda g: -g[3])


def frequencies(lam):
    """omega / (2 pi) = sqrt(lambda) / (2 pi) (band-plot convention)."""
    return [math.sqrt(max(x, 0.0)) / (2.0 * math.pi) for x in lam]


def default_store():
    """The initialised process group's key-value store (atomic add), or None."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return None
    try:
        from torch.distributed import distributed_c10d as c10d
        return c10d._get_default_store()
    except Exception:  # noqa: BLE001 -- no store: fall back to static LPT shares
        return None


_CALLS = [0]   # solve_path calls in this process (all ranks call it alike): store key prefix


class _Locked:
    """Thread-safe iteration over a k index sequence (list or StealQueue)."""

    def __init__(self, it):
        import threading
        self._it = iter(it)
        self._lock = threading.Lock()

    def __iter__(self):
        return self

    def __next__(self):
        with self._lock:
            return next(self._it)


def auto_per_gpu(n):
    """Concurrent solvers per GPU for a grid: the small grids leave the B200
    underfilled (the plane grid of a b = 2 block is 384 CTAs at 64^3), so 2-3
    k-points share it (measured +32 % at 64^3 with 3, +25 % at 96^3 with 2)."""
    pts = int(n[0]) * int(n[1]) * int(n[2])
    return 3 if pts <= 64 ** 3 else (2 if pts <= 96 ** 3 else 1)


def solve_path(a_raw, n, eps, kappas, nev, device=None, checkpoint_dir=None, stream=None, steal=True, per_gpu=1,
               **opts):
    """Band structure along a k-path: every rank (torch.distributed, one
    process per GPU, if initialised) solves its LPT share on its own device
    through the C ABI, stealing unclaimed k from slower ranks when its own
    share is done (``steal``), and the merged, path-ordered records are
    returned on every rank.  ``per_gpu`` > 1 runs that many solvers
    concurrently on the rank's GPU (one host thread and one CUDA stream each;
    the C ABI releases the GIL), which fills the device at small grids
    (2-4 k-points per GPU at 64^3); ``per_gpu="auto"`` picks 3
    up to 64^3 points, 2 up to 96^3, else 1 (measured).  ``eps``:
    (3n,) float64 host array (P:L323-332 layout)."""
    import glob
    import threading

    import torch.distributed as dist

    from . import Lattice, Solver
    rank, world = 0, 1
    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(), dist.get_world_size()
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    lat = Lattice(a_raw, n)
    shares = assign(kappas, world)
    store = default_store() if (steal and world > 1) else None
    _CALLS[0] += 1
    todo = StealQueue(shares, rank, store, prefix="kpath%d" % _CALLS[0]) if store is not None else shares[rank]
    ck = os.path.join(checkpoint_dir, "kpath_rank%d.jsonl" % rank) if checkpoint_dir else None
    others = sorted(glob.glob(os.path.join(checkpoint_dir, "kpath_rank*.jsonl*"))) if checkpoint_dir else []
    meta = run_meta(nev, eps, n=tuple(n), **{k: v for k, v in opts.items()})
    if per_gpu == "auto":
        per_gpu = auto_per_gpu(n)
    if per_gpu <= 1:
        S = Solver(lat, device=device, stream=stream, **opts)
        S.set_epsilon(eps)

        def solve(kap):
            return S.solve(kap, nev, allow_noconv=True)

        recs = run_path(solve, kappas, todo, rank=rank, checkpoint=ck, meta=meta, resume_from=others)
        S.close()
        return gather(recs, len(kappas))
    import torch
    queue = _Locked(todo)
    streams = [torch.cuda.Stream(device=device) for _ in range(per_gpu)]
    solvers = []
    for q in range(per_gpu):
        S = Solver(lat, device=device, stream=streams[q].cuda_stream, **opts)
        S.set_epsilon(eps)
        solvers.append(S)
    results = [[] for _ in range(per_gpu)]
    errors = []

    def worker(q):
        try:
            S = solvers[q]
            results[q] = run_path(lambda kap: S.solve(kap, nev, allow_noconv=True), kappas, queue, rank=rank,
                                  checkpoint=(ck + ".t%d" % q) if ck else None, meta=meta,
                                  resume_from=others)
        except Exception as e:  # noqa: BLE001 -- re-raised below
            errors.append(e)

    th = [threading.Thread(target=worker, args=(q,)) for q in range(per_gpu)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for S in solvers:
        S.close()
    if errors:
        raise errors[0]
    return gather([r for rs in results for r in rs], len(kappas))
