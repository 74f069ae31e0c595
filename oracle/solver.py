"""Oracle: preconditioned conjugate gradients (CG with the multigrid
V-cycle as preconditioner; here, the preconditioner is one
Chebyshev sweep of the smoother from a zero initial guess).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Textbook PCG (Saad, Iterative Methods, Algorithm 9.1), written out step by step:
  r_0 = b - A x_0, z_0 = M r_0, p_0 = z_0
  alpha_k = (r_k, z_k) / (p_k, A p_k)
  x_{k+1} = x_k + alpha_k p_k,  r_{k+1} = r_k - alpha_k A p_k
  stop when ||r_{k+1}|| <= rel_tol ||r_0||
  z_{k+1} = M r_{k+1},  beta_k = (r_{k+1}, z_{k+1}) / (r_k, z_k),  p_{k+1} = z_{k+1} + beta_k p_k
"""
import numpy as np


def pcg(apply_A, apply_M, b, x0, rel_tol=1e-9, max_iter=500):
    """Returns (x, iterations, relative residual)."""
    x = np.array(x0, dtype=np.float64)
    r = b - apply_A(x)
    r0 = np.linalg.norm(r)
    if r0 == 0 or max_iter == 0:
        return x, 0, (1.0 if r0 > 0 else 0.0)
    z = apply_M(r)
    p = z.copy()
    rz = r @ z
    res = 1.0
    k = 0
    for k in range(1, max_iter + 1):
        q = apply_A(p)
        alpha = rz / (p @ q)
        x = x + alpha * p
        r = r - alpha * q
        res = np.linalg.norm(r) / r0
        if res <= rel_tol or k == max_iter:
            break
        z = apply_M(r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, k, res
