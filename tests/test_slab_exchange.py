"""Exchange logic of the slab decomposition (
bnf_solver_create_dist / bnf_opts.slabs) on CPU: world size 2 over gloo.

Each rank holds the Fourier-side j-slab q[k][jl][i] (j = r n2/P + jl) and
runs the z-step of Algorithm 2 on it; the real-space rows are
laid out in the library's block order [q][cl][jl][i] (c = q n3/P + cl) and
exchanged with one all-to-all (torch.distributed, gloo), after which each rank
finishes the y- and x-steps on its z-slab of n3/P whole planes.  The result
must equal the oracle's T q (oracle.fftop.T_apply) on that z-slab; the
reverse path (Algorithm 1, T^*) must return the oracle's T^* p on the j-slab."""
import json
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import fftop, lattice  # noqa: E402
from synthetic import configs  # noqa: E402

N = (8, 6, 4)
KAP = (0.21, -0.37, 0.44)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n1, n2, n3 = N
    P = world
    n2l, n3l = n2 // P, n3 // P
    L = lattice.snap(configs.config(4).a_raw, N)
    D1, D2, D3 = fftop._diag_phases(L, KAP)             # broadcastable over (c|k, b|j, a|i)
    rng = np.random.default_rng(5)
    q_full = rng.standard_normal((n3, n2, n1)) + 1j * rng.standard_normal((n3, n2, n1))
    js = slice(rank * n2l, (rank + 1) * n2l)
    # -------- forward (Algorithm 2): z-step on this j-slab
    x = np.fft.ifft(q_full[:, js, :], axis=0) * n3 * D3[:, js, :]        # [c][jl][i]
    send = np.concatenate([x[qq * n3l:(qq + 1) * n3l] for qq in range(P)])   # [q][cl][jl][i]
    recv = torch.empty(send.size * 2, dtype=torch.float64)
    dist.all_to_all_single(recv, torch.from_numpy(send.view(np.float64).ravel().copy()))
    blocks = recv.numpy().view(np.complex128).reshape(P, n3l, n2l, n1)   # [r][cl][jl][i]
    planes = np.concatenate([blocks[r] for r in range(P)], axis=1)      # [cl][j][i], j = r n2l + jl
    y = np.fft.ifft(planes, axis=1) * n2 * D2
    y = np.fft.ifft(y, axis=2) * n1 * D1
    y /= np.sqrt(n1 * n2 * n3)
    want = fftop.T_apply(L, KAP, q_full)[rank * n3l:(rank + 1) * n3l]
    fwd_err = float(np.abs(y - want).max() / np.abs(want).max())
    # -------- adjoint (Algorithm 1): x- and y-steps on the z-slab, exchange back, z-step on the j-slab
    p_full = rng.standard_normal((n3, n2, n1)) + 1j * rng.standard_normal((n3, n2, n1))
    u = np.fft.fft(p_full[rank * n3l:(rank + 1) * n3l] * np.conj(D1), axis=2)
    u = np.fft.fft(u * np.conj(D2), axis=1)                            # [cl][j][i]
    send = np.concatenate([u[:, r * n2l:(r + 1) * n2l] for r in range(P)])   # [r][cl][jl][i]
    recv = torch.empty(send.size * 2, dtype=torch.float64)
    dist.all_to_all_single(recv, torch.from_numpy(send.view(np.float64).ravel().copy()))
    cols = recv.numpy().view(np.complex128).reshape(P, n3l, n2l, n1)     # [q][cl][jl][i]
    z = np.concatenate([cols[qq] for qq in range(P)], axis=0)          # [c][jl][i]
    z = np.fft.fft(z * np.conj(D3[:, js, :]), axis=0) / np.sqrt(n1 * n2 * n3)
    want_a = fftop.Tstar_apply(L, KAP, p_full)[:, js, :]
    adj_err = float(np.abs(z - want_a).max() / np.abs(want_a).max())
    with open(os.path.join(out_dir, "rank%d.json" % rank), "w") as f:
        json.dump({"fwd": fwd_err, "adj": adj_err}, f)
    dist.barrier()
    dist.destroy_process_group()


def test_slab_all_to_all_world2_gloo(tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        with open(tmp_path / ("rank%d.json" % r)) as f:
            e = json.load(f)
        assert e["fwd"] < 1e-13 and e["adj"] < 1e-13, (r, e)
