"""Oracle: naive element-wise SIPG Laplacian by Gauss quadrature (no sum factorisation).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

What it computes (the plain definition):
for every cell K and test function phi_i (all (p+1)^3 of them),

  y_i = sum_q w_q det J_q (J_q^{-T} grad_xi phi_i) . (J_q^{-T} grad_xi u_h)       Eq. (3)
      + sum_{F in faces(K)} sum_{q in F} dA_q [ sigma_F phi_i (u- - u+)
                                               - phi_i n.(grad u- + grad u+)/2
                                               - (n.grad phi_i)(u- - u+)/2 ]     Eq. (1)

with u_h = sum_j phi_j u_j summed over ALL n^3 functions of the cell (and of the
neighbour for u+), (p+1)^3 Gauss points in the cell and (p+1)^2 on each face
(PAPER.md:201-217), the element-wise arrangement,
  n  = outward unit normal of K = (2s-1) J^{-T} e_d / |J^{-T} e_d|,
  dA = det J |J^{-T} e_d| w_face,
  mirror Dirichlet u+ = -u-, grad u+ = grad u- (reading 4),
  periodic: the neighbour wraps,
  sigma_F = (p+1)^2 * penalty_factor * (A_F/V_K- + A_F/V_K+)/2, A_F and V_K by the
  same Gauss rules; boundary faces use A_F/V_K- (reading 5, pinned
  by tests/test_oracle_brute.py: the Cartesian value (p+1)^2/h, and the documented
  mean on curved interior faces through the single-cell energy identity),
  or, when `user_penalty` (ncells, 6) is given, sigma_F = user_penalty[K, 2d+s]
  (the caller's per-face penalty; equal on both sides of a face).
The neighbour's gradient uses the neighbour's own Jacobian at the shared point.

Dense tables Phi[q][j] = phi_j(xi_q) over all 3D points and functions are library
matmuls (np.einsum) — a primitive step, not a factorisation of the sums.
"""
import numpy as np

from . import basis1d
from .geometry import Mesh


def _tensor_table(rows, deriv_dir=None, drows=None):
    """3D table T[P, J]: product over directions of rows[m][pt_m, j_m] (row of the
    derivative in direction deriv_dir).  Points and functions are lexicographic,
    x fastest.  rows[m] has shape (npts_m, n)."""
    mats = [drows[m] if m == deriv_dir else rows[m] for m in range(3)]
    # kron(z, kron(y, x)) gives index (pz*ny + py)*nx + px for points and functions
    return np.kron(mats[2], np.kron(mats[1], mats[0]))


class SIPG:
    def __init__(self, mesh: Mesh, p: int, basis: str = "hermite", penalty_factor: float = 1.0,
                 user_penalty=None):
        self.mesh, self.p, self.basis, self.pf = mesh, p, basis, penalty_factor
        self.user_penalty = None if user_penalty is None else np.asarray(user_penalty, np.float64).reshape(-1, 6)
        n = self.n = p + 1
        t = basis1d.tables(p, basis)
        self.t = t
        xq, wq = t["xq"], t["wq"]
        # cell tables
        rows = [t["S"]] * 3
        drows = [t["DS"]] * 3
        self.Phi = _tensor_table(rows)
        self.dPhi = [_tensor_table(rows, m, drows) for m in range(3)]
        g = np.stack(np.meshgrid(xq, xq, xq, indexing="ij"), -1)   # [z][y][x] -> need x fastest
        self.xi_cell = np.stack([g[..., 2], g[..., 1], g[..., 0]], -1).reshape(-1, 3)
        # g[iz,iy,ix] = (xq[iz], xq[iy], xq[ix]) so reversed components give (x,y,z)
        self.w_cell = np.kron(wq, np.kron(wq, wq))
        # face tables, keyed (d, s)
        self.face = {}
        for d in range(3):
            for s in (0, 1):
                v = (t["v1"] if s else t["v0"])[None, :]
                dv = (t["d1"] if s else t["d0"])[None, :]
                rows = [v if m == d else t["S"] for m in range(3)]
                drows = [dv if m == d else t["DS"] for m in range(3)]
                Phi = _tensor_table(rows)
                dPhi = [_tensor_table(rows, m, drows) for m in range(3)]
                tang = [m for m in range(3) if m != d]
                pts = np.zeros((n * n, 3))
                a = np.arange(n * n)
                pts[:, tang[0]] = xq[a % n]
                pts[:, tang[1]] = xq[a // n]
                pts[:, d] = float(s)
                w = wq[a % n] * wq[a // n]
                self.face[(d, s)] = (Phi, dPhi, pts, w)
        self._vol = None

    # ---------------------------------------------------------------- geometry
    def volumes(self, cells):
        J = self.mesh.jacobian(cells, self.xi_cell)
        return np.einsum("q,cq->c", self.w_cell, np.linalg.det(J))

    def _face_area_factor(self, J, d, w):
        """dA per face point and J^{-T} e_d: returns (dA, JiT_ed, Jinv)."""
        Jinv = np.linalg.inv(J)
        JiT_ed = Jinv[..., d, :]           # (J^{-T} e_d)_k = (J^{-1})_{d k}
        nrm = np.linalg.norm(JiT_ed, axis=-1)
        dA = np.linalg.det(J) * nrm * w
        return dA, JiT_ed, nrm, Jinv

    def neighbor(self, cells, d, s):
        """Neighbour cell ids across face (d, s); -1 where the face is a mirror boundary."""
        cc = self.mesh.cell_coords(cells).copy()
        cc[:, d] += 2 * s - 1
        N = self.mesh.N[d]
        out = (cc[:, d] < 0) | (cc[:, d] >= N)
        if self.mesh.bc[d] == "periodic":
            cc[:, d] %= N
            nb = self.mesh.cell_id(cc)
        else:
            cc[:, d] = np.clip(cc[:, d], 0, N - 1)
            nb = self.mesh.cell_id(cc)
            nb[out] = -1
        return nb

    # ---------------------------------------------------------------- operator
    def apply(self, u, cells=None, chunk=None):
        """y = A u restricted to the rows of `cells` (default: all cells).

        u: (ndof,) or (ndof, R).  Returns (len(cells)*n^3,) or (len(cells)*n^3, R)."""
        n3 = self.n ** 3
        u = np.asarray(u, dtype=np.float64)
        vec = u.ndim == 1
        U = u.reshape(self.mesh.ncells, n3, -1)
        cells = np.arange(self.mesh.ncells) if cells is None else np.asarray(cells)
        if chunk is None:
            chunk = max(1, int(4e6 // (n3 * 30 * U.shape[2])))
        out = []
        for b in range(0, len(cells), chunk):
            out.append(self._apply_cells(U, cells[b:b + chunk]))
        y = np.concatenate(out, axis=0).reshape(len(cells) * n3, -1)
        return y[:, 0] if vec else y

    def _apply_cells(self, U, cells, own_only=False):
        """own_only: U is (C, n3, R) holding trial functions on `cells` only; every
        other cell's coefficients are zero (used for the diagonal)."""
        p, n = self.p, self.n
        Uc = U if own_only else U[cells]                           # (C, n3, R)
        # ---- cell term, Eq. (3)
        J = self.mesh.jacobian(cells, self.xi_cell)                # (C, Q, 3, 3)
        detJ = np.linalg.det(J)
        Jinv = np.linalg.inv(J)
        gref = np.stack([np.einsum("qj,cjr->cqr", D, Uc) for D in self.dPhi], 2)  # (C,Q,3,R)
        gphys = np.einsum("cqkm,cqkr->cqmr", Jinv, gref)           # J^{-T} g: (J^{-T})_{mk} = Jinv_{km}
        # (J^{-T} grad phi_i).(gphys) = grad phi_i . (J^{-1} gphys)
        t = np.einsum("cqmk,cqkr->cqmr", Jinv, gphys) * (self.w_cell[None, :] * detJ)[..., None, None]
        y = sum(np.einsum("qi,cqr->cir", self.dPhi[m], t[:, :, m]) for m in range(3))
        V = np.einsum("q,cq->c", self.w_cell, detJ)
        # ---- face terms, Eq. (1), element-wise
        for d in range(3):
            for s in (0, 1):
                Phi, dPhi, pts, w = self.face[(d, s)]
                PhiO, dPhiO, ptsO, wO = self.face[(d, 1 - s)]
                Jm = self.mesh.jacobian(cells, pts)                # (C,F,3,3)
                dA, JiT_ed, nrm, Jinv_m = self._face_area_factor(Jm, d, w)
                nvec = (2 * s - 1) * JiT_ed / nrm[..., None]       # outward unit normal
                um = np.einsum("fj,cjr->cfr", Phi, Uc)
                grm = np.stack([np.einsum("fj,cjr->cfr", D, Uc) for D in dPhi], 2)
                gm = np.einsum("cfkm,cfkr->cfmr", Jinv_m, grm)     # J^{-T} grad_xi
                nb = self.neighbor(cells, d, s)
                mirror = nb < 0
                nbc = np.where(mirror, cells, nb)
                if own_only:
                    Un = np.where((nbc == cells)[:, None, None], Uc, 0.0)
                else:
                    Un = U[nbc]
                up = np.einsum("fj,cjr->cfr", PhiO, Un)
                grp = np.stack([np.einsum("fj,cjr->cfr", D, Un) for D in dPhiO], 2)
                Jp = self.mesh.jacobian(nbc, ptsO)
                dAp, _, _, Jinv_p = self._face_area_factor(Jp, d, wO)
                gp = np.einsum("cfkm,cfkr->cfmr", Jinv_p, grp)
                Vp = np.einsum("q,cq->c", self.w_cell, np.linalg.det(self.mesh.jacobian(nbc, self.xi_cell)))
                # mirror principle
                up = np.where(mirror[:, None, None], -um, up)
                gp = np.where(mirror[:, None, None, None], gm, gp)
                AF = dA.sum(1)
                AFp = dAp.sum(1)
                sig_int = 0.5 * (AF / V + AFp / Vp)
                sig = (p + 1) ** 2 * self.pf * np.where(mirror, AF / V, sig_int)
                if self.user_penalty is not None:
                    sig = self.user_penalty[cells, 2 * d + s]
                jump = um - up                                      # (C,F,R)
                avg = 0.5 * np.einsum("cfm,cfmr->cfr", nvec, gm + gp)
                rv = dA[..., None] * (sig[:, None, None] * jump - avg)
                # -(n . J^{-T} grad_xi phi_i) jump/2 dA = grad_xi phi_i . (J^{-1} n) (-jump dA/2)
                cvec = np.einsum("cfmk,cfk->cfm", Jinv_m, nvec)    # J^{-1} n
                rg = -0.5 * (dA[..., None] * jump)[:, :, None, :] * cvec[..., None]
                y += np.einsum("fi,cfr->cir", Phi, rv)
                y += sum(np.einsum("fi,cfr->cir", dPhi[m], rg[:, :, m]) for m in range(3))
        return y                                                     # (C, n3, R)

    def assemble(self):
        """Dense matrix (tiny meshes only): A[:, j] = apply(e_j)."""
        nd = self.mesh.ncells * self.n ** 3
        if nd > 4000:
            raise ValueError("assemble() is for tiny meshes")
        return self.apply(np.eye(nd))

    # ---------------------------------------------------------------- diagonal
    def diagonal(self, cells=None):
        """diag(A) = a(phi_i, phi_i) for every DoF of `cells`: the same element-wise
        form applied to the unit vector e_i, whose neighbours carry zero (mirror
        faces still reflect it).  Returns (len(cells)*n^3,)."""
        n3 = self.n ** 3
        cells = np.arange(self.mesh.ncells) if cells is None else np.asarray(cells)
        E = np.eye(n3)
        chunk = max(1, int(2e6 // (n3 * n3)))
        out = []
        for b in range(0, len(cells), chunk):
            cb = cells[b:b + chunk]
            Uc = np.broadcast_to(E, (len(cb), n3, n3)).copy()
            y = self._apply_cells(Uc, cb, own_only=True)
            out.append(np.einsum("cii->ci", y))
        return np.concatenate(out).reshape(-1)
