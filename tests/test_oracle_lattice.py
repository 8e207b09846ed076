"""Pins for oracle.lattice (§2.2-2.3) against worked examples
(tests/golden/snapping.json) and invariants of eq. (transvec)."""
import json
import math
import os

import numpy as np
import pytest

from oracle import lattice
from synthetic import configs


def _vec(L, deg_in_xy=None, deg_in_xz=None):
    if deg_in_xy is not None:
        t = math.radians(deg_in_xy)
        return [L * math.cos(t), L * math.sin(t), 0.0]
    t = math.radians(deg_in_xz)
    return [L * math.cos(t), 0.0, L * math.sin(t)]


@pytest.fixture(scope="module")
def gold(golden_dir):
    with open(os.path.join(golden_dir, "snapping.json")) as f:
        return json.load(f)


def test_gamma_worked_examples(gold):
    for c in gold["gamma_cases"]:
        a = np.array([[c["L1"], 0, 0], _vec(c["L2"], deg_in_xy=c["gamma_deg"]), [0, 0, 1.0]]).T
        L = lattice.snap(a, (c["n1"], 4, 4))
        assert L.m[0] == c["m1"], c["cite"]
        assert L.cos[0] == pytest.approx(c["cos_gamma"], abs=1e-15), c["cite"]


def test_beta_worked_examples(gold):
    for c in gold["beta_cases"]:
        a = np.array([[c["L1"], 0, 0], [0, 1.0, 0], _vec(c["L3"], deg_in_xz=c["beta_deg"])]).T
        L = lattice.snap(a, (c["n1"], 4, 4))
        assert L.m[1] == c["m2"], c["cite"]
        want = c["cos_beta"] if "cos_beta" in c else eval(c["cos_beta_expr"])
        assert L.cos[1] == pytest.approx(want, abs=1e-15), c["cite"]


def _lattice_for(kind):
    if kind == "fcc_unit":
        s = math.sqrt(2.0)
        return configs.fcc_vectors() * s
    return {"sc": configs.sc_vectors(), "fcc": configs.fcc_vectors(),
            "bcc": configs.bcc_vectors(), "triclinic": configs.triclinic_vectors()}[kind]


def test_lattice_integers(gold):
    for c in gold["lattices"]:
        L = lattice.snap(_lattice_for(c["kind"]), tuple(c["n"]))
        assert L.m == tuple(c["m"]), c["cite"]
        assert L.rho == tuple(c["rho"]), c["cite"]
        if "perm" in c:
            assert L.perm == tuple(c["perm"]), c["cite"]
        if "a" in c:
            np.testing.assert_allclose(L.a, np.array(c["a"]), atol=1e-14, err_msg=c["a_cite"])
        if "alpha_deg" in c:
            assert math.degrees(math.acos(L.cos[2])) == pytest.approx(c["alpha_deg"], abs=5e-5)
        if "angles_deg" in c:
            got = [math.degrees(math.acos(x)) for x in L.cos]
            np.testing.assert_allclose(got, c["angles_deg"], atol=5e-5)


@pytest.mark.parametrize("idx", [1, 2, 3, 4, 5])
def test_transvec_invariants(idx):
    """eq. (transvec): upper triangular, lengths kept, grid alignment
    a2_x = (m1 - rho1 n1) dx, a3_x = (m2 - rho2 n1) dx, a3_y = (m3 - rho3 n2) dy
    (P:L148-211), l = diag(a), delta = l / n."""
    cfg = configs.config(idx)
    L = lattice.snap(cfg.a_raw, cfg.n)
    a = L.a
    assert a[1, 0] == 0 and a[2, 0] == 0 and a[2, 1] == 0
    np.testing.assert_allclose(np.linalg.norm(a, axis=0), L.lengths, rtol=1e-14)
    np.testing.assert_allclose(a, np.diag(L.delta) @ L.Ag, rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(np.diag(a), L.l, rtol=1e-15)
    np.testing.assert_allclose(np.array(L.l) / np.array(L.n), L.delta, rtol=1e-15)
    # cell volume preserved up to the snapping distortion (< 1 %)
    assert abs(np.linalg.det(a) / abs(np.linalg.det(cfg.a_raw)) - 1) < 1e-2


def test_reciprocal_identity():
    """[b]^T [a] = 2 pi I; Omega maps the canonical reciprocal
    basis to the new one; Omega = rotation for an undistorted
    lattice (BCC is not snapped)."""
    for idx in (1, 2, 3, 4):
        cfg = configs.config(idx)
        L = lattice.snap(cfg.a_raw, cfg.n)
        b, om = lattice.reciprocal(L)
        np.testing.assert_allclose(b.T @ L.a, 2 * math.pi * np.eye(3), atol=1e-12)
        bt = 2 * math.pi * np.linalg.inv(L.a_canon).T
        np.testing.assert_allclose(b, om @ bt, atol=1e-12)
    L = lattice.snap(configs.bcc_vectors(), (96, 96, 96))
    _, om = lattice.reciprocal(L)
    np.testing.assert_allclose(om @ om.T, np.eye(3), atol=1e-12)


def test_kvec_reduce_corners():
    """kappa_l = K . a~_l / 2pi: FCC X = (2pi/a)(0,1,0) -> (1/2, 0, 1/2);
    BCC H = (2pi/a)(0,1,0) -> (1/2, -1/2, 1/2)."""
    L = lattice.snap(configs.fcc_vectors(), (12, 12, 12))
    assert lattice.kvec_reduce(L, [0, 2 * math.pi, 0]) == pytest.approx((0.5, 0.0, 0.5))
    L = lattice.snap(configs.bcc_vectors(), (12, 12, 12))
    assert lattice.kvec_reduce(L, [0, 2 * math.pi, 0]) == pytest.approx((0.5, -0.5, 0.5))
    L = lattice.snap(configs.sc_vectors(), (12, 12, 12))
    assert lattice.kvec_reduce(L, configs.config(1).kpoints[0]) == pytest.approx((0.25, 0.15, 0.05))


def test_canonical_relabel_and_rejects():
    L = lattice.snap(configs.triclinic_vectors(), (8, 8, 8))
    assert L.perm == (2, 0, 1) and L.sign3 == 1
    assert lattice.kappa_from_raw(L, (0.1, 0.2, 0.3)) == (0.3, 0.1, 0.2)
    # left-handed input: a3 negated
    a = configs.sc_vectors()
    a[:, 2] *= -1
    L = lattice.snap(a, (4, 4, 4))
    assert L.sign3 == -1
    with pytest.raises(ValueError):
        lattice.snap(configs.sc_vectors(), (0, 4, 4))


def test_gyroid_sampling_bcc():
    """NEXT-2 input: the gyroid of PAPER.md L2402-2407 sampled on the BCC cell
    equals the level set evaluated directly at the Yee points (mapped to the
    original frame), is invariant under the BCC translation (a/2)(1,1,1), and
    fills a plausible fraction of the cell."""
    from synthetic import configs
    from synthetic import eps as E
    a = configs.bcc_vectors()
    n = (12, 12, 12)
    L = lattice.snap(a, n)
    ep = E.sample("gyroid:16", n, L.a, L.delta, L.a_canon)
    inv = np.linalg.inv(L.a)
    for comp in range(3):
        x = E.yee_points(L.delta, n, comp)
        f = x @ inv.T
        f -= np.floor(f)
        X = f @ L.a_canon.T
        want = np.where(E.gyroid_level(X) > 1.1, 16.0, 1.0)
        assert np.array_equal(ep[comp].ravel(), want)
        shifted = E.gyroid_level(X + 0.5)
        np.testing.assert_allclose(shifted, E.gyroid_level(X), atol=1e-12)
    frac = np.mean(np.concatenate([e.ravel() for e in ep]) > 1.0)
    assert 0.02 < frac < 0.3, frac
