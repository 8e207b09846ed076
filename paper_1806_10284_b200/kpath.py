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

    def to_json(self):
        return json.dumps({"index": self.index, "kappa": list(self.kappa), "status": self.status,
                           "lam": list(self.lam), "stats": self.stats, "rank": self.rank,
                           "attempts": self.attempts, "seconds": self.seconds})

    @staticmethod
    def from_json(line):
        d = json.loads(line)
        return KRecord(d["index"], tuple(d["kappa"]), d["status"], d["lam"], d["stats"], d["rank"],
                       d["attempts"], d["seconds"])


def load_checkpoint(path):
    """Finished records of a previous run (status ok or noconv), by k index."""
    done = {}
    if path and os.path.exists(path):
        with open(path) as f:
            for line in f:
                line = line.strip()
                if not line:
                    continue
                try:
                    r = KRecord.from_json(line)
                except (ValueError, KeyError):
                    continue   # torn last line of an interrupted run
                if r.status in ("ok", "noconv"):
                    done[r.index] = r
    return done


def run_path(solve, kappas, indices, rank=0, checkpoint=None, retries=1, clock=time.perf_counter):
    """Solve the k-points ``indices`` (this rank's share) with ``solve``.

    ``solve(kappa)`` returns ``(lam, stats_dict)``; ``stats_dict["rc"]`` may
    mark non-convergence (6 = BNF_ENOCONV).  An exception is retried
    ``retries`` times and then recorded as ``failed`` (the path continues).
    With ``checkpoint`` (a per-rank JSONL path) finished k are skipped and
    new records are appended as they complete."""
    done = load_checkpoint(checkpoint)
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
                    rec = KRecord(i, kap, status, [float(x) for x in lam], dict(st), rank, attempt, clock() - t0)
                    break
                except Exception as e:  # noqa: BLE001 -- recorded, path continues
                    rec = KRecord(i, kap, "failed", [], {"error": str(e)}, rank, attempt, clock() - t0)
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


def frequencies(lam):
    """omega / (2 pi) = sqrt(lambda) / (2 pi) (band-plot convention)."""
    return [math.sqrt(max(x, 0.0)) / (2.0 * math.pi) for x in lam]


def solve_path(a_raw, n, eps, kappas, nev, device=None, checkpoint_dir=None, stream=None, **opts):
    """Band structure along a k-path: every rank (torch.distributed, one
    process per GPU, if initialised) solves its LPT share on its own device
    through the C ABI and the merged, path-ordered records are returned on
    every rank.  ``eps``: (3n,) float64 host array (P:L323-332 layout)."""
    import torch.distributed as dist

    from . import Lattice, Solver
    rank, world = 0, 1
    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(), dist.get_world_size()
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    lat = Lattice(a_raw, n)
    S = Solver(lat, device=device, stream=stream, **opts)
    S.set_epsilon(eps)
    share = assign(kappas, world)[rank]
    ck = os.path.join(checkpoint_dir, "kpath_rank%d.jsonl" % rank) if checkpoint_dir else None

    def solve(kap):
        return S.solve(kap, nev, allow_noconv=True)

    recs = run_path(solve, kappas, share, rank=rank, checkpoint=ck)
    S.close()
    return gather(recs, len(kappas))
