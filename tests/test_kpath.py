"""Host logic of the k-path scheduler (paper_1806_10284_b200/kpath.py):
assignment, retry/checkpoint, and the multi-process gather over gloo
(world_size 2, CPU) -- the N > 1 path of bench.py / solve_path without a GPU."""
import json
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1806_10284_b200 import kpath  # noqa: E402
from synthetic import configs  # noqa: E402


def _fake_solve(kap):
    # deterministic stand-in for Solver.solve: lambda depends only on kappa
    k = np.asarray(kap)
    lam = np.sort(np.abs(np.sin(np.arange(1, 5) * (1.0 + k.sum()))) + 0.1)
    return lam.tolist(), {"rc": 0, "matvecs": 10}


def _path():
    return [tuple(x) for x in configs.config(4).kappa_direct]


def test_assign_covers_every_k_once_and_balances():
    kaps = _path()
    for world in (1, 2, 3, 8):
        share = kpath.assign(kaps, world)
        flat = sorted(i for s in share for i in s)
        assert flat == list(range(len(kaps)))
        costs = [kpath.kpoint_cost(k) for k in kaps]
        loads = [sum(costs[i] for i in s) for s in share]
        assert max(loads) - min(loads) <= max(costs) + 1e-12
        assert share == kpath.assign(kaps, world)   # deterministic


def test_gamma_is_costlier():
    assert kpath.kpoint_cost((0.0, 0.0, 0.0)) > kpath.kpoint_cost((0.1, 0.2, 0.3))
    assert kpath.kpoint_cost((0.5, 0.0, 0.5)) > kpath.kpoint_cost((0.4, 0.1, 0.3))


def test_retry_and_failure_recorded():
    calls = {"n": 0}

    def flaky(kap):
        calls["n"] += 1
        if kap[0] == 0.0 and calls["n"] == 1:
            raise RuntimeError("transient")
        if kap[0] < 0:
            raise RuntimeError("always")
        return _fake_solve(kap)

    kaps = [(0.0, 0.0, 0.0), (-1.0, 0.0, 0.0), (0.2, 0.1, 0.0)]
    recs = kpath.run_path(flaky, kaps, [0, 1, 2], retries=1)
    assert [r.status for r in recs] == ["ok", "failed", "ok"]
    assert recs[0].attempts == 2 and recs[1].attempts == 2


def test_checkpoint_resume_skips_finished(tmp_path):
    kaps = _path()[:6]
    ck = str(tmp_path / "rank0.jsonl")
    first = kpath.run_path(_fake_solve, kaps, [0, 1, 2], checkpoint=ck)
    with open(ck, "a") as f:
        f.write('{"index": 3, "kappa": [')   # torn line of an interrupted run
    seen = []

    def counting(kap):
        seen.append(kap)
        return _fake_solve(kap)

    second = kpath.run_path(counting, kaps, list(range(6)), checkpoint=ck)
    assert len(seen) == 3                                     # only k = 3, 4, 5 solved again
    assert [r.lam for r in second[:3]] == [r.lam for r in first]
    assert [r.index for r in second] == list(range(6))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    kaps = _path()
    share = kpath.assign(kaps, world)[rank]
    recs = kpath.run_path(_fake_solve, kaps, share, rank=rank)
    merged = kpath.gather(recs, len(kaps))
    if rank == 0:
        with open(os.path.join(out_dir, "merged.json"), "w") as f:
            json.dump([[r.index, r.rank, r.lam] for r in merged], f)
    dist.barrier()
    dist.destroy_process_group()


def test_gather_world2_gloo_equals_single_process(tmp_path):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    with open(tmp_path / "merged.json") as f:
        merged = json.load(f)
    kaps = _path()
    single = kpath.merge([kpath.run_path(_fake_solve, kaps, range(len(kaps)))], len(kaps))
    assert [m[0] for m in merged] == list(range(len(kaps)))
    assert {m[1] for m in merged} == {0, 1}                    # both ranks contributed
    for m, s in zip(merged, single):
        assert m[2] == s.lam


def test_frequencies_convention():
    lam = [4 * np.pi ** 2, 0.0]
    assert kpath.frequencies(lam) == [1.0, 0.0]


def test_checkpoint_ignores_other_runs(tmp_path):
    """a checkpoint written with another nev / eps / option set
    (meta) or another kappa for the same index is not reused."""
    kaps = _path()[:4]
    ck = str(tmp_path / "rank0.jsonl")
    kpath.run_path(_fake_solve, kaps, [0, 1, 2, 3], checkpoint=ck, meta="A")
    seen = []

    def counting(kap):
        seen.append(kap)
        return _fake_solve(kap)

    kpath.run_path(counting, kaps, [0, 1, 2, 3], checkpoint=ck, meta="B")
    assert len(seen) == 4                                   # other meta: nothing reused
    seen.clear()
    moved = [kaps[0], (0.9, 0.9, 0.9), kaps[2], kaps[3]]
    kpath.run_path(counting, moved, [0, 1, 2, 3], checkpoint=ck, meta="A")
    assert seen == [(0.9, 0.9, 0.9)]                        # only the changed kappa re-solved
    m1 = kpath.run_meta(16, np.ones(6), block=2)
    assert m1 == kpath.run_meta(16, np.ones(6), block=2)
    assert m1 != kpath.run_meta(16, np.ones(6), block=4) and m1 != kpath.run_meta(10, np.ones(6), block=2)


def test_steal_queue_single_process_covers_all():
    shares = kpath.assign(_path(), 3)
    q = kpath.StealQueue(shares, 1, None)
    got = list(q)
    assert sorted(got) == sorted(i for s in shares for i in s)   # own share, then every other one
    assert got[:len(shares[1])] == shares[1]


def _steal_worker(rank, world, port, out_dir):
    import time
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    kaps = _path()
    shares = kpath.assign(kaps, world)
    q = kpath.StealQueue(shares, rank, kpath.default_store(), prefix="t")

    def slow(kap):        # rank 0 is 20x slower per k: rank 1 must steal from it
        time.sleep(0.2 if rank == 0 else 0.01)
        return _fake_solve(kap)

    recs = kpath.run_path(slow, kaps, q, rank=rank)
    merged = kpath.gather(recs, len(kaps))
    if rank == 0:
        with open(os.path.join(out_dir, "steal.json"), "w") as f:
            json.dump({"merged": [[r.index, r.rank, r.lam] for r in merged],
                       "counts": [sum(1 for r in merged if r.rank == q_) for q_ in range(world)],
                       "shares": shares}, f)
    dist.barrier()
    dist.destroy_process_group()


def test_work_stealing_world2_gloo():
    """World size 2 over gloo: the slow rank's unclaimed k are taken by the
    fast rank; every k is solved exactly once and the merged path equals a
    single-process run."""
    import tempfile
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_steal_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        with open(os.path.join(d, "steal.json")) as f:
            out = json.load(f)
    kaps = _path()
    merged = out["merged"]
    assert [m[0] for m in merged] == list(range(len(kaps)))
    assert out["counts"][1] > len(out["shares"][1])            # rank 1 stole
    single = kpath.merge([kpath.run_path(_fake_solve, kaps, range(len(kaps)))], len(kaps))
    for m, s in zip(merged, single):
        assert m[2] == s.lam


def test_band_gaps():
    """NEXT-2 gap extraction: bands given as lambda = (2 pi omega)^2; a gap
    between bands 1 and 2 (0-based) of width 0.1 in omega / (2 pi)."""
    import math
    om = [[0.25, 0.3, 0.5], [0.15, 0.2, 0.45], [0.12, 0.28, 0.4]]
    recs = [[(2 * math.pi * w) ** 2 for w in o] for o in om]
    g = kpath.band_gaps(recs)
    assert len(g) == 1 and g[0][0] == 1
    assert abs(g[0][1] - 0.3) < 1e-12 and abs(g[0][2] - 0.4) < 1e-12 and abs(g[0][3] - 0.1) < 1e-12


def test_auto_per_gpu():
    assert kpath.auto_per_gpu((12, 12, 12)) == 3 and kpath.auto_per_gpu((64, 64, 64)) == 3
    assert kpath.auto_per_gpu((96, 96, 96)) == 2 and kpath.auto_per_gpu((128, 128, 128)) == 1
