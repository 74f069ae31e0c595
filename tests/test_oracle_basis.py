"""Pins for oracle/basis1d.py against values the paper prints and closed forms.

Every expected value here comes from PAPER.md (cited) or from mathematics
(quadrature exactness, symmetry, partition of unity), never from the CUDA path.
"""
import json
import os

import mpmath as mp

mp.mp.dps = 50  # comparisons in 50 digits, like the oracle's construction
import numpy as np
import pytest
import sympy

from oracle import basis1d as b

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _mp(expr):
    return mp.mpf(str(sympy.N(sympy.sympify(expr), 60)))


@pytest.mark.parametrize("p", [2, 3, 4, 5])
def test_appendix_a_closed_forms(p):
    """Appendix A: coefficients to 1e-12 (SPEC acceptance 1)."""
    gold = _load("appendix_a.json")["basis"][str(p)]
    phis = b.basis_polys(p, "hermite")
    with mp.workdps(50):
        xs = [mp.mpf(k) / 37 for k in range(38)]
        for (scale, roots), phi in zip(gold, phis):
            ref = b.Poly.from_roots(_mp(scale), [_mp(r) for r in roots])
            assert len(ref.c) == len(phi.c)
            for a_, r_ in zip(phi.c, ref.c):
                assert abs(a_ - r_) < 1e-12 * max(1, abs(r_))
            for x in xs:
                assert abs(phi(x) - ref(x)) < 1e-12


def test_p3_constants():
    """xi_1 = 2/7, alpha_0 = -7/2, alpha_1 = 11/2."""
    _, prm = b.hermite_like(3)
    assert abs(prm["xi1"] - mp.mpf(2) / 7) < 1e-40
    assert abs(prm["alpha0"] + mp.mpf(7) / 2) < 1e-40
    assert abs(prm["alpha1"] - mp.mpf(11) / 2) < 1e-40


def test_p2_alpha1():
    """alpha_1 = 2 for p=2: D_f = [-2, 2, 0] at xi=0."""
    t = b.tables(2)
    np.testing.assert_allclose(t["d0"], [-2, 2, 0], atol=1e-14)


def test_fig2_p7_rounded():
    """Figure 2, p=7: scales rounded to integers, roots to ~3 digits."""
    gold = _load("fig2_p7.json")["basis"]
    phis = b.basis_polys(7, "hermite")
    for (scale, roots), phi in zip(gold, phis):
        lead = float(phi.c[-1])
        assert abs(lead - scale) <= 0.5 + 1e-9, (lead, scale)
        r = np.sort(np.roots([float(c) for c in reversed(phi.c)]).real)
        np.testing.assert_allclose(r, np.sort(roots), atol=1.5e-3)


def test_condition_table():
    """tab:condition_mass to the printed 3 significant digits."""
    g = _load("tab_condition_mass.json")
    for p, h, gl in zip(g["p"], g["hermite_like"], g["gauss_lobatto"]):
        assert abs(b.mass_condition(p, "hermite") - h) <= 0.05 + 1e-12
        tol = 0.005 if gl < 10 else 0.05
        assert abs(b.mass_condition(p, "gl") - gl) <= tol + 1e-12


@pytest.mark.parametrize("p", range(1, 9))
@pytest.mark.parametrize("basis", ["hermite", "gl"])
def test_partition_of_unity_and_symmetry(p, basis):
    """sum_i phi_i = 1 and phi_i(xi) = phi_{p-i}(1-xi)."""
    phis = b.basis_polys(p, basis)
    with mp.workdps(50):
        for k in range(23):
            x = mp.mpf(k) / 22 + mp.mpf(1) / 97
            assert abs(mp.fsum(f(x) for f in phis) - 1) < 1e-40
            for i in range(p + 1):
                assert abs(phis[i](x) - phis[p - i](1 - x)) < 1e-40


@pytest.mark.parametrize("p", range(1, 9))
def test_hermite_face_sparsity(p):
    """S_f = [1,0..0], D_f = [-a, a, 0..0] at xi=0, mirrored at 1 (Eq. (9)):
    only two 1D functions have a nonzero value or derivative at each end."""
    t = b.tables(p)
    assert abs(t["v0"][0] - 1) < 1e-15 and np.all(np.abs(t["v0"][1:]) < 1e-30)
    assert abs(t["d0"][0] + t["d0"][1]) < 1e-13 * abs(t["d0"][1])
    assert np.all(np.abs(t["d0"][2:]) < 1e-30)
    assert abs(t["v1"][-1] - 1) < 1e-15 and np.all(np.abs(t["v1"][:-1]) < 1e-30)
    np.testing.assert_allclose(t["d1"][::-1], -t["d0"], rtol=1e-14, atol=1e-30)


@pytest.mark.parametrize("p", range(3, 9))
def test_orthogonality_phi0_phi1_and_bubbles(p):
    """int phi_0 phi_1 = 0 and L2-orthogonal bubbles."""
    M = b.mass_matrix_mp(p, "hermite")
    assert abs(M[0, 1]) < 1e-40
    for i in range(2, p - 1):
        for j in range(2, p - 1):
            if i != j:
                assert abs(M[i, j]) < 1e-40


def test_jacobi_roots():
    """P^{4,4}_1 root 1/2; P^{4,4}_2 roots 1/2 -+ sqrt(1/44) (Appendix A p=5)."""
    assert abs(b.jacobi44_roots(1)[0] - mp.mpf(1) / 2) < 1e-45
    r = b.jacobi44_roots(2)
    assert abs(r[0] - (mp.mpf(1) / 2 - mp.sqrt(mp.mpf(1) / 44))) < 1e-40
    assert abs(r[1] - (mp.mpf(1) / 2 + mp.sqrt(mp.mpf(1) / 44))) < 1e-40
    r3 = b.jacobi44_roots(3)
    assert abs(r3[1] - mp.mpf(1) / 2) < 1e-40 and abs(r3[0] + r3[2] - 1) < 1e-40


@pytest.mark.parametrize("n", range(1, 10))
def test_gauss_rule_exactness(n):
    """n-point Gauss on (0,1): weights sum to 1, exact for xi^k, k <= 2n-1."""
    x, w = b.gauss_legendre(n)
    with mp.workdps(50):
        for k in range(2 * n):
            assert abs(mp.fsum(wi * xi ** k for xi, wi in zip(x, w)) - mp.mpf(1) / (k + 1)) < 1e-40
    if n == 2:
        assert abs(x[0] - (mp.mpf(1) / 2 - 1 / (2 * mp.sqrt(3)))) < 1e-40


def test_gauss_lobatto_points():
    """GL(3) on [0,1] = {0, 1/2, 1}; GL(n) nodes symmetric."""
    x = b.gauss_lobatto_points(3)
    assert [float(v) for v in x] == [0.0, 0.5, 1.0]
    for n in range(2, 10):
        x = b.gauss_lobatto_points(n)
        for i in range(n):
            assert abs(x[i] + x[n - 1 - i] - 1) < 1e-40


def test_p1_is_lagrange_and_gl_agrees():
    """p=1 Hermite-like = {1-xi, xi} = GL p=1."""
    for basis in ("hermite", "gl"):
        phis = b.basis_polys(1, basis)
        assert [float(c) for c in phis[0].c] == [1.0, -1.0]
        assert [float(c) for c in phis[1].c] == [0.0, 1.0]


@pytest.mark.parametrize("p", range(1, 9))
def test_change_matrix(p):
    """T[i][j] = phi_j(x_i^GL): rows sum to 1, T[0] = e_0, T^{-1}T = I; T applied to the
    Hermite coefficients of a degree-p polynomial gives its GL nodal values."""
    T, Ti = b.change_matrix(p)
    n = p + 1
    np.testing.assert_allclose(T.sum(1), 1.0, atol=1e-14)
    np.testing.assert_allclose(T[0], np.eye(n)[0], atol=1e-15)
    np.testing.assert_allclose(Ti @ T, np.eye(n), atol=1e-13)
    # coefficients of f by interpolation at the Gauss points (S c = f(xq))
    t = b.tables(p)
    rng = np.random.default_rng(p)
    a = rng.standard_normal(n)
    f = lambda x: np.polyval(a, x)
    c = np.linalg.solve(t["S"], f(t["xq"]))
    xgl = np.array([float(v) for v in b.gauss_lobatto_points(n)])
    np.testing.assert_allclose(T @ c, f(xgl), rtol=1e-12, atol=1e-12)
    if p == 2:
        np.testing.assert_allclose(T, [[1, 0, 0], [0.25, 0.5, 0.25], [0, 0, 1]], atol=1e-16)


@pytest.mark.parametrize("p", range(1, 9))
def test_tables_consistent_with_polynomials(p):
    """S and DS tables are the basis and its derivative at the Gauss points; S is invertible
    and S^{-1} reproduces xi exactly (linear reproduction)."""
    t = b.tables(p)
    c = np.linalg.solve(t["S"], t["xq"])
    # the interpolant of xi has derivative 1 everywhere
    np.testing.assert_allclose(t["DS"] @ c, 1.0, atol=1e-12)
    np.testing.assert_allclose(t["DS"].sum(1), 0.0, atol=1e-11)
