"""Independent pins of the oracle's GEOMETRY handling (oracle/sipg.py), the parts the
Cartesian pins cannot see: the J^{-T} metric of Eq. (3) on non-diagonal
Jacobians, the face normals and areas of Eq. (1) on affine and curved
cells, and the penalty convention on curved interior faces (reading R5).

Nothing here uses oracle/sipg.py's arithmetic or oracle/geometry.py's Jacobian; every
reference is built from the definitions:
  * the mesh map x(xi) written out from the configuration text (PAPER.md:788-797 for the
    paper's affine brick, BASELINE.json C3 for the curved map) and differentiated
    NUMERICALLY in 40-digit mpmath (central differences), not from an analytic Jacobian;
  * physical gradients from the linear system J^T g = grad_xi phi (the chain rule), not
    from an explicit inverse-transpose product;
  * face areas and normals from the tangent cross product (J e_t1) x (J e_t2), not from
    Nanson's formula det J |J^{-T} e_d|;
  * the bilinear form written FACE-WISE as the symmetric SIPG form
    sigma [[v]][[u]] - [[v]] {{d_n u}} - {{d_n v}} [[u]] (mirror faces: 2 sigma v u -
    v d_n u - u d_n v, reading R4), not the oracle's element-wise arrangement;
  * SIPG consistency: for an affine map and u a bubble of the undeformed unit-box
    coordinates, A u = (int phi_i f)_i with f = -Laplace_x u evaluated by mpmath finite
    differences of u(x) in PHYSICAL coordinates (u(x) through the inverse affine map).
Each test below fails for the classic mistakes J^{-1} <-> J^{-T} (metric or normal),
a dropped face term, a wrong normal sign and max-instead-of-mean penalties; see
tools/oracle_mutants.py, which runs these tests against such mutants of oracle/sipg.py.
"""
import itertools

import mpmath as mp
import numpy as np
import pytest

from oracle import basis1d
from oracle.geometry import Mesh
from oracle.sipg import SIPG

DPS = 40
PAPER_BRICK = dict(L=(1.12, 0.24, 0.36, 0.24, 1.36, 0.48, 0.36, 0.48, 1.60),
                   lo=(-0.95, -0.9, -0.85), hi=(0.95, 0.89, 0.83))
SKEW = dict(L=(1.0, 0.45, -0.2, -0.3, 0.9, 0.35, 0.15, -0.4, 1.1), lo=(0.0, 0.0, 0.0), hi=(1.0, 0.8, 1.2))


# ---------------------------------------------------------------- the map, from its definition
def map_point(geo, N, cell, xi):
    """x(xi) on cell (cx,cy,cz): X = lo + (c + xi) h, x = L X, then (curved) x_i += amp
    sin(2 pi Xh_j) sin(2 pi Xh_k) with (i,j,k) cyclic and Xh = (c + xi)/N the unit-box
    coordinate (BASELINE.json C3 wording; reading R6).  mpmath in, mpmath out."""
    L = geo.get("L", (1, 0, 0, 0, 1, 0, 0, 0, 1))
    lo = geo.get("lo", (0, 0, 0))
    hi = geo.get("hi", (1, 1, 1))
    amp = geo.get("amp", 0.0)
    X = [mp.mpf(lo[m]) + (cell[m] + xi[m]) * (mp.mpf(hi[m]) - mp.mpf(lo[m])) / N[m] for m in range(3)]
    x = [sum(mp.mpf(L[3 * i + m]) * X[m] for m in range(3)) for i in range(3)]
    if amp:
        Xh = [(cell[m] + xi[m]) / mp.mpf(N[m]) for m in range(3)]
        s = [mp.sin(2 * mp.pi * v) for v in Xh]
        for i in range(3):
            j, k = (i + 1) % 3, (i + 2) % 3
            x[i] += mp.mpf(amp) * s[j] * s[k]
    return x


def jac_numeric(geo, N, cell, xi):
    """J[i][m] = d x_i / d xi_m by 4th-order central differences at 40 digits."""
    eps = mp.mpf(10) ** -9
    J = mp.matrix(3, 3)
    for m in range(3):
        cols = []
        for sgn in (2, 1, -1, -2):
            pt = list(xi)
            pt[m] = pt[m] + sgn * eps
            cols.append(map_point(geo, N, cell, pt))
        for i in range(3):
            J[i, m] = (-cols[0][i] + 8 * cols[1][i] - 8 * cols[2][i] + cols[3][i]) / (12 * eps)
    return J


def _cell_coords(N, c):
    return (c % N[0], (c // N[0]) % N[1], c // (N[0] * N[1]))


class Geo:
    """Quadrature-point geometry of every cell, from the numerically differentiated map."""

    def __init__(self, geo, N, p):
        self.geo, self.N, self.p = geo, N, p
        self.n = n = p + 1
        t = basis1d.tables(p)
        self.t = t
        with mp.workdps(DPS):
            xq = [mp.mpf(v) for v in t["xq"]]
            self.xq = xq
            self.nc = N[0] * N[1] * N[2]
            self.cell = {}
            for c in range(self.nc):
                cc = _cell_coords(N, c)
                dets, Js = [], []
                for qz, qy, qx in itertools.product(range(n), repeat=3):
                    J = jac_numeric(geo, N, cc, (xq[qx], xq[qy], xq[qz]))
                    Js.append(J)
                    dets.append(mp.det(J))
                w = np.array([t["wq"][qx] * t["wq"][qy] * t["wq"][qz]
                              for qz, qy, qx in itertools.product(range(n), repeat=3)])
                V = float(sum(mp.mpf(w[q]) * dets[q] for q in range(len(dets))))
                self.cell[c] = (Js, dets, w, V)

    def face_points(self, c, d, s):
        """(J at the face points, area weights dA = |J e_t1 x J e_t2| w, outward unit normals)
        for face (d, s) of cell c; points ordered (a over t1 fastest, b over t2)."""
        n, t = self.n, self.t
        t1, t2 = [m for m in range(3) if m != d]
        cc = _cell_coords(self.N, c)
        out = []
        with mp.workdps(DPS):
            for b in range(n):
                for a in range(n):
                    xi = [None] * 3
                    xi[d] = mp.mpf(s)
                    xi[t1] = self.xq[a]
                    xi[t2] = self.xq[b]
                    J = jac_numeric(self.geo, self.N, cc, xi)
                    e1 = [J[i, t1] for i in range(3)]
                    e2 = [J[i, t2] for i in range(3)]
                    cr = [e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                          e1[0] * e2[1] - e1[1] * e2[0]]
                    area = mp.sqrt(sum(v * v for v in cr))
                    nv = [v / area for v in cr]
                    # orient outward: along +J e_d for s = 1, against it for s = 0
                    ed = [J[i, d] for i in range(3)]
                    if (sum(nv[i] * ed[i] for i in range(3)) > 0) != (s == 1):
                        nv = [-v for v in nv]
                    w = t["wq"][a] * t["wq"][b]
                    out.append((J, float(area) * w, np.array([float(v) for v in nv])))
        return out


def phys_grad(J, gref):
    """Solve J^T g = grad_xi (the chain rule d/dxi_m = sum_i dx_i/dxi_m d/dx_i) for every
    column of gref (3, k); float64 result."""
    Jt = np.array([[float(J[i, m]) for i in range(3)] for m in range(3)])   # Jt[m][i] = J[i][m]
    return np.linalg.solve(Jt, gref)


def _basis_at(t, xi_pts):
    """(values (P, n3), reference gradients (P, 3, n3)) of all tensor-product functions."""
    p = len(t["xq"]) - 1
    n = p + 1
    vals, grads = [], []
    for xi in xi_pts:
        V, D = basis1d.eval_basis(p, "hermite", [float(v) for v in xi])   # (3, n): row m at xi_m
        f = np.einsum("k,j,i->kji", V[2], V[1], V[0]).reshape(-1)
        gx = np.einsum("k,j,i->kji", V[2], V[1], D[0]).reshape(-1)
        gy = np.einsum("k,j,i->kji", V[2], D[1], V[0]).reshape(-1)
        gz = np.einsum("k,j,i->kji", D[2], V[1], V[0]).reshape(-1)
        vals.append(f)
        grads.append(np.stack([gx, gy, gz]))
    del n
    return np.array(vals), np.array(grads)


def brute_force_matrix(geo, N, p, bc):
    """Dense SIPG matrix, face-wise symmetric form, geometry from the numerically
    differentiated map.  Cell-wise DoF order, lexicographic x fastest (R9)."""
    G = Geo(geo, N, p)
    n = p + 1
    n3 = n ** 3
    nc = G.nc
    A = np.zeros((nc * n3, nc * n3))
    xq = [float(v) for v in G.t["xq"]]
    cell_xi = [(xq[qx], xq[qy], xq[qz]) for qz, qy, qx in itertools.product(range(n), repeat=3)]
    Vc, Gc = _basis_at(G.t, cell_xi)
    # ---- cell terms: sum_q w_q det J (grad_x phi_i . grad_x phi_j)
    for c in range(nc):
        Js, dets, w, _ = G.cell[c]
        blk = np.zeros((n3, n3))
        for q in range(len(Js)):
            g = phys_grad(Js[q], Gc[q])               # (3, n3)
            blk += w[q] * float(dets[q]) * (g.T @ g)
        A[c * n3:(c + 1) * n3, c * n3:(c + 1) * n3] += blk
    # ---- faces
    pen = (p + 1) ** 2

    def face_data(c, d, s):
        pts = G.face_points(c, d, s)
        t1, t2 = [m for m in range(3) if m != d]
        xis = []
        for b in range(n):
            for a in range(n):
                xi = [0.0] * 3
                xi[d], xi[t1], xi[t2] = float(s), xq[a], xq[b]
                xis.append(xi)
        V, Gr = _basis_at(G.t, xis)
        return pts, V, Gr

    for d in range(3):
        for c in range(nc):
            cc = list(_cell_coords(N, c))
            # face (d, s=1) of c: interior (periodic or not last) or mirror
            for s in (0, 1):
                nb = list(cc)
                nb[d] += 1 if s else -1
                inside = 0 <= nb[d] < N[d]
                if bc[d] == "periodic":
                    nb[d] %= N[d]
                    inside = True
                if inside and s == 0:
                    continue                     # interior faces once, from the lower cell
                pts, V, Gr = face_data(c, d, s)
                AF = sum(dA for _, dA, _ in pts)
                if not inside:                    # mirror face: 2 sigma v u - v dn u - u dn v
                    sig = pen * AF / G.cell[c][3]
                    blk = np.zeros((n3, n3))
                    for q, (J, dA, nv) in enumerate(pts):
                        dn = nv @ phys_grad(J, Gr[q])
                        v = V[q]
                        blk += dA * (2 * sig * np.outer(v, v) - np.outer(v, dn) - np.outer(dn, v))
                    A[c * n3:(c + 1) * n3, c * n3:(c + 1) * n3] += blk
                    continue
                cn = nb[0] + N[0] * (nb[1] + N[1] * nb[2])
                pts_n, Vn, Grn = face_data(cn, d, 1 - s)
                sig = pen * 0.5 * (AF / G.cell[c][3] + AF / G.cell[cn][3])
                # jump [[w]] = w(c) - w(cn) with n the outward normal of c
                for q, (J, dA, nv) in enumerate(pts):
                    Jn = pts_n[q][0]
                    jm = np.concatenate([V[q], -Vn[q]])
                    dnm = 0.5 * np.concatenate([nv @ phys_grad(J, Gr[q]), nv @ phys_grad(Jn, Grn[q])])
                    blk = dA * (sig * np.outer(jm, jm) - np.outer(jm, dnm) - np.outer(dnm, jm))
                    idx = np.concatenate([np.arange(c * n3, (c + 1) * n3), np.arange(cn * n3, (cn + 1) * n3)])
                    A[np.ix_(idx, idx)] += blk
    return A


BRUTE_CASES = [
    ("paper_affine", PAPER_BRICK, (1, 1, 1), ("dirichlet",) * 3, 1),
    ("paper_affine", PAPER_BRICK, (2, 1, 1), ("dirichlet",) * 3, 2),
    ("skew_affine", SKEW, (2, 1, 1), ("periodic", "dirichlet", "dirichlet"), 2),
    ("curved", dict(amp=0.05), (1, 1, 1), ("dirichlet",) * 3, 2),
    ("curved", dict(amp=0.05), (2, 1, 1), ("dirichlet",) * 3, 2),
    ("curved_periodic", dict(amp=0.05), (2, 1, 1), ("periodic", "dirichlet", "dirichlet"), 1),
    ("cartesian", dict(lo=(0, 0, 0), hi=(1.5, 0.5, 0.75)), (2, 1, 1), ("dirichlet",) * 3, 2),
]


@pytest.mark.parametrize("name,geo,N,bc,p", BRUTE_CASES, ids=[f"{c[0]}-{c[2][0]}x1x1-p{c[4]}" for c in BRUTE_CASES])
def test_oracle_equals_brute_force_bilinear_form(name, geo, N, bc, p):
    """SURVEY.md §8(c) 'matvec (brute force)': mpmath geometry, dense face-wise bilinear form
    on 1x1x1 and 2x1x1 meshes (Cartesian, the paper's affine brick, a skewed affine map and
    the C3 curved map), same Gauss rules as the oracle."""
    ref = brute_force_matrix(geo, N, p, bc)
    m = Mesh(N=N, lo=geo.get("lo", (0, 0, 0)), hi=geo.get("hi", (1, 1, 1)),
             L=geo.get("L", (1, 0, 0, 0, 1, 0, 0, 0, 1)), amp=geo.get("amp", 0.0), bc=bc)
    A = SIPG(m, p).assemble()
    assert np.abs(A - ref).max() <= 1e-11 * np.abs(ref).max()


# ---------------------------------------------------------------- SIPG consistency, affine maps
def _bubble_coeffs(p, N):
    """Hermite coefficients of Xh(1-Xh) on N cells (interpolation at the Gauss points)."""
    t = basis1d.tables(p)
    out = []
    for c in range(N):
        x = (c + t["xq"]) / N
        out.append(np.linalg.solve(t["S"], x * (1 - x)))
    return np.array(out)                    # (N, n)


@pytest.mark.parametrize("geo", [PAPER_BRICK, SKEW], ids=["paper_brick", "skew"])
@pytest.mark.parametrize("p", [2, 3])
def test_affine_bubble_consistency(geo, p):
    """u(x) = b(Xh(x)), b = prod_m Xh_m (1 - Xh_m) with Xh the unit-box coordinate of the
    undeformed mesh: u is in the discrete space on every affine cell and vanishes on the
    boundary, so SIPG consistency plus exact Gauss quadrature give A u = (int_K phi_i f)_i,
    f = -Laplace_x u.  f is evaluated by 40-digit finite differences of u in PHYSICAL
    coordinates, u(x) through the inverse of the affine map x = L (lo + Xh (hi - lo))."""
    N = (2, 2, 2)
    n = p + 1
    lo, hi, Lm = geo["lo"], geo["hi"], geo["L"]
    m = Mesh(N=N, lo=lo, hi=hi, L=Lm)
    op = SIPG(m, p)
    B = [_bubble_coeffs(p, N[d]) for d in range(3)]
    U = np.einsum("ai,bj,ck->cbakji", B[0], B[1], B[2]).reshape(-1)
    y = op.apply(U)
    t = basis1d.tables(p)
    with mp.workdps(DPS):
        Lmp = mp.matrix(3, 3)
        for i in range(3):
            for k in range(3):
                Lmp[i, k] = mp.mpf(Lm[3 * i + k])
        Linv = Lmp ** -1
        ext = [mp.mpf(hi[k]) - mp.mpf(lo[k]) for k in range(3)]

        def u_of_x(x):
            X = Linv * mp.matrix(x)
            Xh = [(X[k] - mp.mpf(lo[k])) / ext[k] for k in range(3)]
            r = mp.mpf(1)
            for v in Xh:
                r *= v * (1 - v)
            return r

        def f_of_x(x):
            eps = mp.mpf(10) ** -8
            u0 = u_of_x(x)
            lap = 0
            for i in range(3):
                xp = list(x)
                xm = list(x)
                xp[i] += eps
                xm[i] -= eps
                lap += (u_of_x(xp) - 2 * u0 + u_of_x(xm)) / eps ** 2
            return -lap

        ref = np.zeros_like(y).reshape(-1, n ** 3)
        for c in range(m.ncells):
            cc = _cell_coords(N, c)
            # |det J| of the affine cell from the numerically differentiated map
            detJ = float(mp.det(jac_numeric(geo, N, cc, (mp.mpf(0.5),) * 3)))
            fq = []
            for qz, qy, qx in itertools.product(range(n), repeat=3):
                xi = (mp.mpf(t["xq"][qx]), mp.mpf(t["xq"][qy]), mp.mpf(t["xq"][qz]))
                fq.append(float(f_of_x(map_point(geo, N, cc, xi))))
            fq = np.array(fq)
            w = np.einsum("k,j,i->kji", t["wq"], t["wq"], t["wq"]).reshape(-1)
            Phi = np.einsum("ck,bj,ai->cbakji", t["S"], t["S"], t["S"]).reshape(n ** 3, n ** 3)  # [q][i]
            ref[c] = detJ * (Phi.T @ (w * fq))
    ref = ref.reshape(-1)
    assert np.abs(y - ref).max() <= 1e-10 * np.abs(ref).max()


# ---------------------------------------------------------------- penalty convention (R5)
@pytest.mark.parametrize("p", [1, 2])
def test_single_cell_energy_identity_curved(p):
    """u = 1 on one cell K, 0 elsewhere: the cell term and every gradient term vanish
    (grad u = 0 on both sides; sum_i grad phi_i = 0), so
        1_K^T A 1_K = sum_{interior F of K} sigma_F A_F + sum_{mirror F of K} 2 sigma_F A_F,
    sigma_F = (p+1)^2 (A_F/V_K + A_F/V_K')/2 on interior faces, (p+1)^2 A_F/V_K on mirror
    faces (R5), A_F from tangent cross products, V_K = sum_q w_q det J_q with J
    numerically differentiated.  The centre cell of a 3x3x3 curved mesh has six interior
    faces with six different neighbour volumes; a corner cell mixes both kinds."""
    N = (3, 3, 3)
    geo = dict(amp=0.05)
    G = Geo(geo, N, p)
    m = Mesh(N=N, amp=0.05)
    op = SIPG(m, p)
    n3 = (p + 1) ** 3
    pen = (p + 1) ** 2
    for c in (13, 0):
        e = np.zeros(m.ncells * n3)
        e[c * n3:(c + 1) * n3] = 1.0
        lhs = e @ op.apply(e)
        cc = _cell_coords(N, c)
        rhs = 0.0
        for d in range(3):
            for s in (0, 1):
                AF = sum(dA for _, dA, _ in G.face_points(c, d, s))
                nb = list(cc)
                nb[d] += 1 if s else -1
                if 0 <= nb[d] < N[d]:
                    cn = nb[0] + N[0] * (nb[1] + N[1] * nb[2])
                    rhs += pen * 0.5 * (AF / G.cell[c][3] + AF / G.cell[cn][3]) * AF
                else:
                    rhs += 2 * pen * AF / G.cell[c][3] * AF
        assert abs(lhs - rhs) <= 1e-12 * rhs, (c, lhs, rhs)
