"""Oracle: basis change, GL-Jacobi preconditioner and the Chebyshev smoother.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

basis_change (reading 11): v = T^{x3} u with
  T[i][j] = phi_j^H(x_i^GL), i.e. v_i = u_h(x_i^GL) = the nodal Gauss-Lobatto values
  of the Hermite-like expansion, obtained by evaluating all n^3 functions at all
  n^3 GL nodes (dense table, no factorisation).  The inverse / transposes use the
  dense kron(T,T,T) with numpy.linalg.solve.

pinv (Eq. (12), reading 13):
  P^{-1} r = (T^{-1})^{x3} diag(A_GL)^{-1} (T^{-T})^{x3} r,
  diag(A_GL) the point-Jacobi diagonal of the same operator in the nodal GL basis
  (PAPER.md:1795-1798), computed by oracle.sipg.SIPG(..., basis="gl").diagonal().

chebyshev (Eq. (11); recurrence of SPEC.md:432, reading 14):
  [alpha, beta] = [lo, hi] * lambda_max, c = (beta+alpha)/2, delta = (beta-alpha)/2
  u_1 = u_0 + (1/c) P^{-1}(b - A u_0)
  sigma_1 = c/delta, rho_1 = 1/sigma_1, rho_{j+1} = 1/(2 sigma_1 - rho_j)
  u_{j+1} = u_j + rho_{j+1} rho_j (u_j - u_{j-1}) + (2 rho_{j+1}/delta) P^{-1}(b - A u_j)
  "degree k" = k applications of A.
"""
import numpy as np

from . import basis1d


def T3(p: int):
    T, _ = basis1d.change_matrix(p)
    return np.kron(T, np.kron(T, T))


def basis_change(p: int, u, op: str = "T"):
    """Apply B^{x3} per cell for B in {T, Tinv, TT (T^T), TinvT (T^{-T})}."""
    n3 = (p + 1) ** 3
    U = np.asarray(u, dtype=np.float64).reshape(-1, n3)
    if op == "T":
        # v_i = u_h(x_i^GL): evaluate every Hermite function at every GL node
        V, _ = basis1d.eval_basis(p, "hermite", basis1d.gauss_lobatto_points(p + 1))
        E = np.kron(V, np.kron(V, V))          # E[node, function]
        return (U @ E.T).reshape(-1)
    A = T3(p)
    if op == "TT":
        return (U @ A).reshape(-1)
    if op == "Tinv":
        return np.linalg.solve(A, U.T).T.reshape(-1)
    if op == "TinvT":
        return np.linalg.solve(A.T, U.T).T.reshape(-1)
    raise ValueError(op)


class GLJacobi:
    """P^{-1} of Eq. (12) with the Gauss-Lobatto point-Jacobi diagonal."""

    def __init__(self, sipg_gl):
        self.p = sipg_gl.p
        self.dinv = 1.0 / sipg_gl.diagonal()

    def __call__(self, r):
        z = basis_change(self.p, r, "TinvT")
        z = z * self.dinv
        return basis_change(self.p, z, "Tinv")


class PointJacobi:
    """P = diag(A) in the working basis."""

    def __init__(self, sipg):
        self.dinv = 1.0 / sipg.diagonal()

    def __call__(self, r):
        return r * self.dinv


def chebyshev(apply_A, apply_Pinv, b, x0, degree, lambda_max, lo=0.06, hi=1.2):
    """Chebyshev iteration of Eq. (11); returns u_degree."""
    alpha, beta = lo * lambda_max, hi * lambda_max
    if not (0 < alpha < beta):
        raise ValueError("need 0 < lo*lambda_max < hi*lambda_max")
    c = 0.5 * (beta + alpha)
    delta = 0.5 * (beta - alpha)
    u_prev = np.array(x0, dtype=np.float64)
    if degree == 0:
        return u_prev
    u = u_prev + (1.0 / c) * apply_Pinv(b - apply_A(u_prev))
    sigma1 = c / delta
    rho = 1.0 / sigma1
    for _ in range(1, degree):
        rho_new = 1.0 / (2.0 * sigma1 - rho)
        u_next = u + rho_new * rho * (u - u_prev) + (2.0 * rho_new / delta) * apply_Pinv(b - apply_A(u))
        u_prev, u, rho = u, u_next, rho_new
    return u


def lanczos_lambda_max(apply_A, apply_Pinv, n, iters=15):
    """Largest Ritz value of P^{-1}A after `iters` Lanczos steps from the start
    vector [-5.5, -4.5, ..., 5.5] repeated, in the
    P-inner product (P^{-1}A is P-self-adjoint)."""
    v = np.tile(np.arange(-5.5, 6.0, 1.0), n // 12 + 1)[:n].astype(np.float64)
    # work with w = P^{-1} r:  inner product <x, y>_P = x . P y  ->  use r-space
    z = apply_Pinv(v)
    beta = np.sqrt(v @ z)
    v_prev = np.zeros(n)
    z_prev = np.zeros(n)
    v, z = v / beta, z / beta
    alphas, betas = [], []
    b_prev = 0.0
    for _ in range(iters):
        w = apply_A(z)                     # A z, z = P^{-1} v
        a = w @ z
        w = w - a * v - b_prev * v_prev
        wz = apply_Pinv(w)
        b = np.sqrt(max(w @ wz, 0.0))
        alphas.append(a)
        if b < 1e-300:
            break
        betas.append(b)
        v_prev, z_prev = v, z
        v, z = w / b, wz / b
        b_prev = b
    k = len(alphas)
    Tm = np.diag(alphas) + np.diag(betas[:k - 1], 1) + np.diag(betas[:k - 1], -1)
    return float(np.linalg.eigvalsh(Tm)[-1])
