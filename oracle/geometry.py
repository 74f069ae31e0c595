"""Oracle: the analytic mesh map x(xi) of a structured hex mesh and its Jacobian.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Reading:
  undeformed   X_m = lo_m + (c_m + xi_m) h_m,   h_m = (hi_m - lo_m)/N_m
  unit box     Xh_m = (c_m + xi_m)/N_m
  map          x_i = sum_m L_im X_m + amp * sin(2 pi Xh_j) sin(2 pi Xh_k),
               (i, j, k) cyclic
  Jacobian     J_im = dx_i/dxi_m = L_im h_m
                      + amp * (2 pi / N_m) * d/dXh_m [sin(2 pi Xh_j) sin(2 pi Xh_k)]
The Jacobian is analytic (not finite differences, not isoparametric).
"""
from dataclasses import dataclass

import numpy as np


@dataclass
class Mesh:
    N: tuple                       # cells per direction (Nx, Ny, Nz), z slowest
    lo: tuple = (0.0, 0.0, 0.0)
    hi: tuple = (1.0, 1.0, 1.0)
    L: tuple = (1.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0)
    amp: float = 0.0
    bc: tuple = ("dirichlet", "dirichlet", "dirichlet")
    inv_jac: np.ndarray = None     # optional per-cell J^{-1} (ncells, 3, 3): affine cells

    @property
    def h(self):
        return np.array([(self.hi[m] - self.lo[m]) / self.N[m] for m in range(3)])

    @property
    def ncells(self):
        return int(self.N[0] * self.N[1] * self.N[2])

    def cell_coords(self, cells):
        """(cx, cy, cz) of lexicographic cell ids (x fastest, z slowest)."""
        cells = np.asarray(cells)
        cx = cells % self.N[0]
        cy = (cells // self.N[0]) % self.N[1]
        cz = cells // (self.N[0] * self.N[1])
        return np.stack([cx, cy, cz], axis=-1)

    def cell_id(self, cc):
        return cc[..., 0] + self.N[0] * (cc[..., 1] + self.N[1] * cc[..., 2])

    def jacobian(self, cells, xi):
        """J at reference points xi (P,3) of each cell: shape (C, P, 3, 3)."""
        cc = self.cell_coords(cells).astype(np.float64)       # (C,3)
        xi = np.asarray(xi, dtype=np.float64)                  # (P,3)
        C, P = cc.shape[0], xi.shape[0]
        if self.inv_jac is not None:
            Ji = self.inv_jac[np.asarray(cells)]
            J = np.linalg.inv(Ji)
            return np.broadcast_to(J[:, None], (C, P, 3, 3)).copy()
        L = np.array(self.L, dtype=np.float64).reshape(3, 3)
        h = self.h
        J = np.empty((C, P, 3, 3))
        J[:] = L * h[None, :]                                  # L_im h_m
        if self.amp != 0.0:
            N = np.array(self.N, dtype=np.float64)
            Xh = (cc[:, None, :] + xi[None, :, :]) / N         # (C,P,3)
            s = np.sin(2 * np.pi * Xh)
            co = np.cos(2 * np.pi * Xh)
            for i in range(3):
                j, k = (i + 1) % 3, (i + 2) % 3
                J[:, :, i, j] += self.amp * 2 * np.pi / N[j] * co[..., j] * s[..., k]
                J[:, :, i, k] += self.amp * 2 * np.pi / N[k] * s[..., j] * co[..., k]
        return J

    def position(self, cells, xi):
        """Physical points x (C, P, 3) (used by tests that integrate functions)."""
        cc = self.cell_coords(cells).astype(np.float64)
        xi = np.asarray(xi, dtype=np.float64)
        lo = np.array(self.lo)
        h = self.h
        X = lo + (cc[:, None, :] + xi[None, :, :]) * h
        L = np.array(self.L, dtype=np.float64).reshape(3, 3)
        x = np.einsum("im,cpm->cpi", L, X)
        if self.amp != 0.0:
            N = np.array(self.N, dtype=np.float64)
            Xh = (cc[:, None, :] + xi[None, :, :]) / N
            s = np.sin(2 * np.pi * Xh)
            for i in range(3):
                j, k = (i + 1) % 3, (i + 2) % 3
                x[..., i] += self.amp * s[..., j] * s[..., k]
        return x


def mesh_from_spec(spec) -> Mesh:
    """Oracle mesh from a synthetic.MeshSpec (plain data)."""
    return Mesh(N=tuple(spec.n_cells), lo=tuple(spec.box_lo), hi=tuple(spec.box_hi),
                L=tuple(spec.linear_map), amp=float(spec.deform_amp), bc=tuple(spec.bc))
