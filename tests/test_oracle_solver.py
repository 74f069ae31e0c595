"""Pins of the PCG oracle (oracle/solver.py) against a dense solve, and of the Lanczos
estimate against the dense generalized eigenvalue problem, on tiny meshes."""
import numpy as np
import pytest
import scipy.linalg

from oracle import smoother as sm
from oracle import solver
from oracle.geometry import mesh_from_spec
from oracle.sipg import SIPG
from synthetic import MeshSpec, uniform_vector


@pytest.mark.parametrize("inner", ["gl_jacobi", "point_jacobi"])
def test_pcg_converges_to_dense_solve(inner):
    spec = MeshSpec(degree=3, n_cells=(2, 2, 3), seed=5)
    om = mesh_from_spec(spec)
    H = SIPG(om, 3)
    A = H.assemble()
    b = uniform_vector(spec.n_dofs, 9)
    P = sm.GLJacobi(SIPG(om, 3, "gl")) if inner == "gl_jacobi" else sm.PointJacobi(H)
    lmax = sm.lanczos_lambda_max(H.apply, P, spec.n_dofs)
    M = lambda r: sm.chebyshev(H.apply, P, r, np.zeros_like(r), 3, lmax)   # noqa: E731
    x, it, res = solver.pcg(H.apply, M, b, np.zeros_like(b), rel_tol=1e-11, max_iter=200)
    xs = np.linalg.solve(A, b)
    assert res <= 1e-11
    assert np.linalg.norm(x - xs) <= 1e-9 * np.linalg.norm(xs)
    assert it < (60 if inner == "gl_jacobi" else 200)   # point Jacobi in the Hermite basis is slow


def test_pcg_identity_preconditioner_is_cg_in_n_steps():
    """Exact arithmetic CG terminates in at most n steps (here: a tiny SPD system)."""
    rng = np.random.default_rng(0)
    Q = rng.standard_normal((12, 12))
    A = Q @ Q.T + 12 * np.eye(12)
    b = rng.standard_normal(12)
    x, it, res = solver.pcg(lambda v: A @ v, lambda r: r, b, np.zeros(12), rel_tol=1e-13, max_iter=40)
    assert it <= 14 and res <= 1e-13
    assert np.allclose(A @ x, b, atol=1e-10)


def test_lanczos_below_and_near_true_lambda_max():
    spec = MeshSpec(degree=3, n_cells=(2, 2, 2), seed=5)
    om = mesh_from_spec(spec)
    H = SIPG(om, 3)
    A = H.assemble()
    P = sm.GLJacobi(SIPG(om, 3, "gl"))
    Pinv = np.stack([P(e) for e in np.eye(spec.n_dofs)], 1)
    lam_true = scipy.linalg.eigh(A, np.linalg.inv(Pinv), eigvals_only=True)[-1]
    est = sm.lanczos_lambda_max(H.apply, P, spec.n_dofs, iters=15)
    assert est <= lam_true * (1 + 1e-12)
    assert est >= 0.97 * lam_true
