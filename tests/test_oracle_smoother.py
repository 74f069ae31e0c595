"""Pins for oracle/smoother.py: basis change, GL-Jacobi, Chebyshev recurrence.

References: the closed-form Chebyshev polynomial, exact fixed
points, and the cross-basis equivalence that defines Eq. (12)'s purpose
("the same iteration counts as the nodal Gauss-Lobatto basis").
"""
import numpy as np
import pytest

from oracle import basis1d
from oracle.geometry import Mesh
from oracle.sipg import SIPG
from oracle import smoother as sm


def _cheb_T(k, x):
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    inside = np.abs(x) <= 1
    out[inside] = np.cos(k * np.arccos(x[inside]))
    xo = x[~inside]
    out[~inside] = np.sign(xo) ** k * np.cosh(k * np.arccosh(np.abs(xo)))
    return out


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_chebyshev_closed_form(k):
    """A = diag(lambda), P = I, b = 0: e_k = T_k((b+a-2l)/(b-a)) / T_k((b+a)/(b-a)) e_0."""
    lam = np.linspace(0.01, 2.5, 20)
    lmax = 2.4
    a, b = 0.06 * lmax, 1.2 * lmax
    u = sm.chebyshev(lambda x: lam * x, lambda r: r, np.zeros(20), np.ones(20), k, lmax)
    ref = _cheb_T(k, (b + a - 2 * lam) / (b - a)) / _cheb_T(k, np.array([(b + a) / (b - a)]))[0]
    np.testing.assert_allclose(u, ref, rtol=1e-12, atol=1e-14)


def test_chebyshev_fixed_point():
    m = Mesh(N=(2, 2, 2))
    op = SIPG(m, 2)
    A = op.assemble()
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, A.shape[0])
    b = A @ x
    P = sm.PointJacobi(op)
    u = sm.chebyshev(op.apply, P, b, x, 5, 2.0)
    np.testing.assert_allclose(u, x, atol=1e-13)


def test_chebyshev_cross_basis_equivalence():
    """Hermite + (T^-1 D_GL^-1 T^-T) smoothing == GL point-Jacobi smoothing mapped by T:
    with b_GL = T^-T b_H and u_GL0 = T u_H0, u_H = T^-1 u_GL after every step."""
    p = 3
    m = Mesh(N=(2, 2, 2), amp=0.05)
    H, G = SIPG(m, p), SIPG(m, p, "gl")
    rng = np.random.default_rng(1)
    nd = m.ncells * (p + 1) ** 3
    bH, uH0 = rng.uniform(-1, 1, nd), rng.uniform(-1, 1, nd)
    lmax = 2.6
    uH = sm.chebyshev(H.apply, sm.GLJacobi(G), bH, uH0, 5, lmax)
    bG = sm.basis_change(p, bH, "TinvT")
    uG0 = sm.basis_change(p, uH0, "T")
    uG = sm.chebyshev(G.apply, sm.PointJacobi(G), bG, uG0, 5, lmax)
    np.testing.assert_allclose(uH, sm.basis_change(p, uG, "Tinv"), rtol=1e-11, atol=1e-11)


def test_lanczos_diagonal():
    """A = diag(1..20), P = I: 15 Lanczos steps estimate lambda_max in [19.5, 20]
    (SPEC.md:425)."""
    lam = np.arange(1.0, 21.0)
    est = sm.lanczos_lambda_max(lambda x: lam * x, lambda r: r, 20, 15)
    assert 19.5 <= est <= 20.0 + 1e-12


def test_lanczos_gl_jacobi_lambda_max():
    """P^{-1}A for the Hermite basis with the GL-Jacobi P has the spectrum of D_GL^{-1} A_GL."""
    p = 3
    m = Mesh(N=(3, 3, 3))
    H, G = SIPG(m, p), SIPG(m, p, "gl")
    AG = G.assemble()
    true = np.max(np.linalg.eigvals(AG / np.diag(AG)[:, None]).real)
    est = sm.lanczos_lambda_max(H.apply, sm.GLJacobi(G), m.ncells * (p + 1) ** 3, 15)
    assert 0.97 * true <= est <= true * (1 + 1e-12)


@pytest.mark.parametrize("p", [1, 2, 5, 8])
def test_basis_change_ops(p):
    """T^{x3}: evaluation at the GL nodes; Tinv inverts it; TT and TinvT are the adjoints."""
    n3 = (p + 1) ** 3
    rng = np.random.default_rng(p)
    u = rng.uniform(-1, 1, 3 * n3)
    v = rng.uniform(-1, 1, 3 * n3)
    Tu = sm.basis_change(p, u, "T")
    np.testing.assert_allclose(sm.basis_change(p, Tu, "Tinv"), u, atol=1e-12)
    assert abs(Tu @ v - u @ sm.basis_change(p, v, "TT")) < 1e-12 * n3
    Tiu = sm.basis_change(p, u, "Tinv")
    assert abs(Tiu @ v - u @ sm.basis_change(p, v, "TinvT")) < 1e-11 * n3
    # values at GL nodes of a tensor polynomial given by its coefficients
    T, _ = basis1d.change_matrix(p)
    np.testing.assert_allclose(Tu[:n3], np.kron(T, np.kron(T, T)) @ u[:n3], atol=1e-13)
    if p == 1:
        np.testing.assert_allclose(Tu, u, atol=1e-15)
