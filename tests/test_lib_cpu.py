"""CPU-side checks of the C-ABI library (no GPU compute): it loads, exports
every symbol include/bnf.h declares, its host lattice setup is bit-equal
to the oracle's (T0 of SURVEY §4), and the solver refuses to run without a
CUDA device (no CPU fallback)."""
import math
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bnf():
    import paper_1806_10284_b200 as m
    return m


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "bnf.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:int|void|char)\s*\*?\s*(bnf_\w+)\s*\(", txt, re.M)))


def test_exports_every_header_symbol(bnf):
    syms = _header_symbols()
    assert len(syms) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", bnf.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (bnf_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert sorted(bnf.EXPORTS) == syms
    assert bnf.version() == 1


def test_library_is_sm100a(bnf):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", bnf.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("idx", [1, 2, 3, 4, 5])
def test_lattice_bit_equal_to_oracle(bnf, idx):
    from oracle import lattice as olat
    from synthetic import configs
    cfg = configs.config(idx)
    L = bnf.Lattice(cfg.a_raw, cfg.n)
    O = olat.snap(cfg.a_raw, cfg.n)
    assert L.m == O.m and L.rho == O.rho and L.perm == O.perm and L.sign3 == O.sign3
    assert np.array_equal(L.Ag, O.Ag)
    np.testing.assert_allclose(L.a, O.a, rtol=0, atol=1e-15)
    np.testing.assert_allclose(L.delta, O.delta, rtol=1e-15)
    if cfg.kappa_direct is None:
        for K in cfg.kpoints[:5]:
            np.testing.assert_allclose(L.kvec_reduce(K), olat.kvec_reduce(O, K), atol=1e-15)


@pytest.mark.parametrize("idx", [1, 2, 3, 4])
def test_yee_points(bnf, idx):
    """bnf_yee_points (P:L323-332 edge midpoints): the snapped-frame points are
    ((a+h1)dx, (b+h2)dy, (c+h3)dz) x-fastest; the original-frame points are the
    wrapped fractional coordinates in the snapped cell applied to a_canon --
    the map the synthetic eps sampler uses, so sampling the shapes at them
    reproduces the sampler's eps field exactly."""
    from synthetic import configs, eps as E
    cfg = configs.config(idx)
    n = cfg.n if idx < 4 else (16, 12, 10)
    L = bnf.Lattice(cfg.a_raw, n)
    inv = np.linalg.inv(L.a)
    for comp in range(3):
        xs = L.yee_points(comp, bnf.FRAME_SNAPPED)
        np.testing.assert_array_equal(xs, E.yee_points(L.delta, n, comp))
        f = xs @ inv.T
        f -= np.floor(f)
        xo = L.yee_points(comp, bnf.FRAME_ORIGINAL)
        # same fractional coordinates modulo the lattice (a point on a cell face may wrap to
        # either side, depending on the last bit of its coordinate), inside the canonical cell
        g = np.linalg.solve(L.a_canon, xo.T).T
        assert g.min() > -1e-12 and g.max() < 1 + 1e-12
        d = g - f
        assert np.abs(d - np.round(d)).max() <= 1e-12
    if cfg.shape != "noise42":
        e_s = E.sample(cfg.shape, n, L.a, L.delta, L.a_canon)[1].ravel()
        inside = E._inside(L.yee_points(1, bnf.FRAME_ORIGINAL), cfg.shape, L.a_canon)
        np.testing.assert_array_equal(np.where(inside, E.EPS_IN, E.EPS_OUT), e_s)
    with pytest.raises(bnf.BnfError):
        L.yee_points(3)


def test_lattice_random_bit_equal(bnf):
    from oracle import lattice as olat
    from tests.test_oracle_curl import random_lattices
    from synthetic import configs
    rng = np.random.default_rng(99)
    count = 0
    while count < 200:
        try:
            a = configs.triclinic_vectors(1.0, rng.uniform(0.6, 1), rng.uniform(0.6, 1), *rng.uniform(50, 130, 3))
        except ValueError:
            continue
        a = a[:, rng.permutation(3)] * rng.uniform(0.5, 2.0)
        n = tuple(int(x) for x in rng.integers(3, 40, 3))
        try:
            O = olat.snap(a, n)
        except ValueError:
            with pytest.raises(bnf.BnfError):
                bnf.Lattice(a, n)
            continue
        L = bnf.Lattice(a, n)
        assert (L.m, L.rho, L.perm, L.sign3) == (O.m, O.rho, O.perm, O.sign3)
        count += 1


def test_lattice_errors(bnf):
    from synthetic import configs
    with pytest.raises(bnf.BnfError) as e:
        bnf.Lattice(configs.sc_vectors(), (0, 4, 4))
    assert e.value.code == bnf.EINVAL


def test_host_herm_eig_matches_numpy(bnf):
    rng = np.random.default_rng(3)
    for n in (1, 2, 5, 17, 60):
        a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        a = a + a.conj().T
        w, z = bnf.host_herm_eig(a)
        np.testing.assert_allclose(w, np.linalg.eigvalsh(a), atol=1e-12 * max(1, np.abs(w).max()))
        np.testing.assert_allclose(a @ z, z * w[None, :], atol=1e-11 * max(1, np.abs(w).max()))
        np.testing.assert_allclose(z.conj().T @ z, np.eye(n), atol=1e-12)
    # degenerate spectrum
    q, _ = np.linalg.qr(rng.standard_normal((8, 8)) + 1j * rng.standard_normal((8, 8)))
    a = q @ np.diag([1, 1, 1, 2, 2, 3, 3, 3.0]) @ q.conj().T
    w, z = bnf.host_herm_eig(a)
    np.testing.assert_allclose(w, [1, 1, 1, 2, 2, 3, 3, 3], atol=1e-12)


def test_solver_refuses_without_gpu(bnf):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from synthetic import configs
    L = bnf.Lattice(configs.sc_vectors(), (4, 4, 4))
    with pytest.raises(bnf.BnfError) as e:
        bnf.Solver(L)
    assert e.value.code == bnf.ECUDA


@pytest.mark.parametrize("idx", [1, 4, 5])
def test_kappa_canonical_equals_oracle(bnf, idx):
    """bnf_kappa_canonical (the ABI's raw -> canonical relabel, R10) equals the
    oracle's kappa_from_raw on the configs whose k are given as raw kappa
    (config 4: cyclic relabel; 5: FCC) and on a left-handed cell (sign flip)."""
    from oracle import lattice as olat
    from synthetic import configs
    cfg = configs.config(idx)
    cases = [(cfg.a_raw, cfg.n)]
    lh = cfg.a_raw.copy()
    lh[:, [0, 1]] = lh[:, [1, 0]]          # swap two vectors: left-handed raw triple
    cases.append((lh, cfg.n))
    rng = np.random.default_rng(idx)
    for a, n in cases:
        L = bnf.Lattice(a, n)
        O = olat.snap(a, n)
        assert L.perm == O.perm and L.sign3 == O.sign3
        for _ in range(5):
            kr = rng.uniform(-1, 1, 3)
            assert L.kappa_from_raw(kr) == olat.kappa_from_raw(O, kr)
