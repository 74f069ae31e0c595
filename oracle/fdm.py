"""Oracle: fast-diagonalisation (FDM) block-Jacobi preconditioner.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The steps in the paper's order (Section "Choice of inner preconditioner for Hermite-like
basis", Eqs. (13)-(15)):

1. 1D matrices of an *interior* element of length h (the cell term
   factorises as in Eq. (13); "proceeding similarly with the face integrals"):
     M[i][j]    = h * int_0^1 phi_i phi_j
     L_DG[i][j] = (1/h) int_0^1 phi_i' phi_j'
                  + sum over the two end points of the element-wise SIPG face terms of
                    Eq. (1) with the neighbour set to zero:
                    sigma phi_i phi_j - (phi_i dn phi_j + dn phi_i phi_j) / 2,
     sigma = (p+1)^2 / h, dn = n d/dx = (+-1/h) d/dxi.
   Integrals by the (p+1)-point Gauss rule (exact for these polynomial degrees).
2. A^(K) = M (x) M (x) L_DG + M (x) L_DG (x) M + L_DG (x) M (x) M   (Eq. (14)); with one
   h per direction for anisotropic cells (the paper's form when h_x = h_y = h_z).
3. The generalized symmetric definite eigenproblem L_DG z = lambda M z (library routine
   scipy.linalg.eigh, normalised Z^T M Z = I); T = column-wise concatenation of the z.
4. P_d^-1 = (I (x) I (x) Lambda + I (x) Lambda (x) I + Lambda (x) I (x) I)^-1   (Eq. (15)).
5. P^-1 r = Z^{(x)3} P_d^-1 (Z^T)^{(x)3} r on every cell: Eq. (12) read with T = Z^T
   (reading R19), the orientation that makes P^-1 the exact inverse of A^(K),
   which is the property the paper states for this block-Jacobi preconditioner.  The
   interior-element matrices are used for every cell, boundary cells included
   (PAPER.md:2160-2163).
"""
import numpy as np
import scipy.linalg

from . import basis1d


def interior_1d(p: int, h: float, basis: str = "hermite", penalty_factor: float = 1.0):
    """(L_DG, M) of one interior element of length h (step 1)."""
    t = basis1d.tables(p, basis)
    S, DS, w = t["S"], t["DS"], t["wq"]
    M = h * (S.T * w) @ S
    L = (DS.T * w) @ DS / h
    sigma = penalty_factor * (p + 1) ** 2 / h
    for v, d, nrm in ((t["v0"], t["d0"], -1.0), (t["v1"], t["d1"], 1.0)):
        dn = nrm * d / h                      # outward normal derivative at this end
        L += sigma * np.outer(v, v) - 0.5 * (np.outer(v, dn) + np.outer(dn, v))
    return L, M


def cell_matrix(p: int, h, basis: str = "hermite", penalty_factor: float = 1.0):
    """A^(K) of Eq. (14); h = (h_x, h_y, h_z).  DoF order x fastest (kron(z, kron(y, x)))."""
    (Lx, Mx), (Ly, My), (Lz, Mz) = (interior_1d(p, hd, basis, penalty_factor) for hd in h)
    return (np.kron(Mz, np.kron(My, Lx)) + np.kron(Mz, np.kron(Ly, Mx)) + np.kron(Lz, np.kron(My, Mx)))


class FDM:
    """P^-1 of the FDM block-Jacobi preconditioner (steps 3-5) for cells of size h."""

    def __init__(self, p: int, h, basis: str = "hermite", penalty_factor: float = 1.0):
        self.p = p
        self.Z, self.lam = [], []
        for hd in h:
            L, M = interior_1d(p, hd, basis, penalty_factor)
            lam, Z = scipy.linalg.eigh(L, M)          # L Z = M Z diag(lam), Z^T M Z = I
            self.Z.append(Z)
            self.lam.append(lam)
        lx, ly, lz = self.lam
        # Eq. (15), index (k, j, i) with i (x) fastest
        self.dinv = 1.0 / (lz[:, None, None] + ly[None, :, None] + lx[None, None, :])
        Zx, Zy, Zz = self.Z
        self.Zf = np.kron(Zz, np.kron(Zy, Zx))          # Z^{(x)3}

    def __call__(self, r):
        n3 = (self.p + 1) ** 3
        R = np.asarray(r, dtype=np.float64).reshape(-1, n3)
        w = R @ self.Zf                                  # (Z^T)^{(x)3} r, per cell (row)
        w = w * self.dinv.reshape(-1)
        return (w @ self.Zf.T).reshape(-1)
