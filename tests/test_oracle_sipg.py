"""Pins for oracle/sipg.py (the naive element-wise SIPG quadrature).

Independent references used here (none of them is the oracle's own code path):
  * an independent 1D SIPG assembly written FACE-WISE (interior-face jumps and
    averages) and combined by the Kronecker sum of Eq. (14)
    (PAPER.md:2141-2143), which holds on Cartesian meshes;
  * closed forms of the continuous bilinear form for polynomials the discrete
    space reproduces exactly (SIPG consistency + exact Gauss quadrature);
  * the Laplace eigenvalue 3 pi^2 of the unit cube;
  * structural invariants: symmetry, positive definiteness (mirror), constants in
    the nullspace (periodic), the basis-independence A_H = T3^T A_GL T3
    (PAPER.md:127-129), and Nanson-free face areas from tangent cross products.
"""
import numpy as np
import pytest

from oracle import basis1d
from oracle.geometry import Mesh
from oracle.sipg import SIPG
from oracle import smoother as sm


# ---------------------------------------------------------------- 1D reference
def sipg_1d(p, N, lo, hi, bc, basis="hermite"):
    """Global 1D SIPG matrix L and mass M on N cells of [lo, hi], assembled face by face:
    sum_K int v'u' + sum_F sigma [v][u] - [v]{u'} - {v'}[u], sigma = (p+1)^2/h,
    mirror faces: u+ = -u-, u'+ = u'- (PAPER.md:150-174)."""
    t = basis1d.tables(p, basis)
    n = p + 1
    h = (hi - lo) / N
    w, S, DS = t["wq"], t["S"], t["DS"]
    Mloc = h * (S.T * w) @ S
    Kloc = (DS.T * w) @ DS / h
    nd = N * n
    L = np.zeros((nd, nd))
    M = np.zeros((nd, nd))
    for c in range(N):
        sl = slice(c * n, (c + 1) * n)
        L[sl, sl] += Kloc
        M[sl, sl] += Mloc
    sig = (p + 1) ** 2 / h
    # trace vectors of one cell at its left (0) and right (1) end, physical derivative
    val = {0: t["v0"], 1: t["v1"]}
    der = {0: t["d0"] / h, 1: t["d1"] / h}

    def add(ci, si, cj, sj, coef_vu):
        L[ci * n:(ci + 1) * n, cj * n:(cj + 1) * n] += coef_vu

    for f in range(N + 1):
        left, right = f - 1, f          # cells sharing the face at x_f
        if bc == "periodic":
            left %= N
            right %= N
            if f == N:
                continue
        if 0 <= left < N and 0 <= right < N and (bc == "periodic" or 0 < f < N):
            # interior face, normal +1 from left to right: [w] = w_left - w_right
            jl, jr = val[1], -val[0]            # jump coefficients
            al, ar = 0.5 * der[1], 0.5 * der[0]  # average of derivatives
            for (ci, jv, av) in ((left, jl, al), (right, jr, ar)):
                for (cj, ju, au) in ((left, jl, al), (right, jr, ar)):
                    add(ci, 0, cj, 0, sig * np.outer(jv, ju) - np.outer(jv, au) - np.outer(av, ju))
        else:
            # mirror boundary face of cell c with outward normal nu: jump 2u, avg nu*u'
            c, s, nu = (right, 0, -1.0) if f == 0 else (left, 1, 1.0)
            v, d = val[s], der[s]
            add(c, s, c, s, 2 * sig * np.outer(v, v) - nu * np.outer(v, d) - nu * np.outer(d, v))
    return L, M


def kron_sum_3d(p, Ncells, lo, hi, bc, basis="hermite"):
    """Eq. (14): A = M_z (x) M_y (x) L_x + M_z (x) L_y (x) M_x + L_z (x) M_y (x) M_x,
    reordered from direction-global to cell-wise lexicographic DoF order."""
    n = p + 1
    Ls, Ms = [], []
    for d in range(3):
        L, M = sipg_1d(p, Ncells[d], lo[d], hi[d], bc[d], basis)
        Ls.append(L)
        Ms.append(M)
    A = (np.kron(Ms[2], np.kron(Ms[1], Ls[0])) + np.kron(Ms[2], np.kron(Ls[1], Ms[0]))
         + np.kron(Ls[2], np.kron(Ms[1], Ms[0])))
    # global index in direction-major order: gz*(NY*NX) + gy*NX + gx, g = c*n + i
    Nx, Ny, Nz = Ncells
    perm = np.empty(A.shape[0], dtype=np.int64)
    k = 0
    for cz in range(Nz):
        for cy in range(Ny):
            for cx in range(Nx):
                for iz in range(n):
                    for iy in range(n):
                        for ix in range(n):
                            gx, gy, gz = cx * n + ix, cy * n + iy, cz * n + iz
                            perm[k] = (gz * Ny * n + gy) * Nx * n + gx
                            k += 1
    return A[np.ix_(perm, perm)]


@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("bc", ["dirichlet", "periodic"])
def test_cartesian_equals_kronecker_sum(p, bc):
    N = (3, 2, 2)
    lo, hi = (0.0, -0.5, 0.25), (1.5, 0.5, 1.0)     # anisotropic cells catch swapped axes
    m = Mesh(N=N, lo=lo, hi=hi, bc=(bc,) * 3)
    A = SIPG(m, p).assemble()
    K = kron_sum_3d(p, N, lo, hi, (bc,) * 3)
    assert np.abs(A - K).max() <= 1e-13 * np.abs(K).max()


def test_cartesian_mixed_bc_gl_basis():
    N = (2, 3, 2)
    bc = ("dirichlet", "periodic", "dirichlet")
    m = Mesh(N=N, bc=bc)
    A = SIPG(m, 3, "gl").assemble()
    K = kron_sum_3d(3, N, (0, 0, 0), (1, 1, 1), bc, "gl")
    assert np.abs(A - K).max() <= 1e-13 * np.abs(K).max()


# ---------------------------------------------------------------- closed forms
def _interp_coeffs(p, f1d, N):
    """Hermite coefficients of a univariate polynomial of degree <= p on N cells of [0,1]."""
    t = basis1d.tables(p)
    out = []
    for c in range(N):
        x = (c + t["xq"]) / N
        out.append(np.linalg.solve(t["S"], f1d(x)))
    return np.concatenate(out)       # direction-global order


def _tensor_field(p, N, fx, fy, fz):
    """Cell-wise coefficient vector of fx(x) fy(y) fz(z)."""
    n = p + 1
    cx, cy, cz = (_interp_coeffs(p, f, N).reshape(N, n) for f in (fx, fy, fz))
    U = np.einsum("ai,bj,ck->cbakji", cx, cy, cz)      # [cz,cy,cx,iz,iy,ix]
    return U.reshape(-1)


@pytest.mark.parametrize("p,N", [(2, 2), (3, 4), (4, 2), (5, 2)])
def test_closed_forms_unit_cube(p, N):
    """[0,1]^3, N^3 cells, mirror Dirichlet:
       1'A1 = 12 N (p+1)^2 (only the boundary penalty 2 sigma |F| survives, 6 faces),
       x'Ax = 14 sigma/3 - 1 with sigma = (p+1)^2 N,
       u_b = x(1-x)y(1-y)z(1-z): 1'A u_b = int -Lap u_b = 1/6, u_b'A u_b = int |grad u_b|^2 = 1/900."""
    m = Mesh(N=(N, N, N))
    op = SIPG(m, p)
    one = np.ones(m.ncells * (p + 1) ** 3)
    A1 = op.apply(one)
    assert abs(one @ A1 - 12 * N * (p + 1) ** 2) < 1e-9 * 12 * N * (p + 1) ** 2
    x = _tensor_field(p, N, lambda s: s, np.ones_like, np.ones_like)
    sig = (p + 1) ** 2 * N
    assert abs(x @ op.apply(x) - (14 * sig / 3 - 1)) < 1e-10 * sig
    q = lambda s: s * (1 - s)
    ub = _tensor_field(p, N, q, q, q)
    Aub = op.apply(ub)
    assert abs(one @ Aub - 1 / 6) < 1e-12
    assert abs(ub @ Aub - 1 / 900) < 1e-13


@pytest.mark.parametrize("p", [2, 3])
def test_consistency_A_ub_equals_M_f(p):
    """SIPG consistency: A u_b = M f entrywise with f = -Lap u_b (Gauss exact on Cartesian)."""
    N = 3
    m = Mesh(N=(N, N, N))
    op = SIPG(m, p)
    q = lambda s: s * (1 - s)
    two = lambda s: 2.0 * np.ones_like(s)
    one = np.ones_like
    ub = _tensor_field(p, N, q, q, q)
    f = (_tensor_field(p, N, two, q, q) + _tensor_field(p, N, q, two, q)
         + _tensor_field(p, N, q, q, two))
    t = basis1d.tables(p)
    h = 1.0 / N
    Mloc = h * (t["S"].T * t["wq"]) @ t["S"]
    M3 = np.kron(Mloc, np.kron(Mloc, Mloc))
    Mf = (f.reshape(-1, (p + 1) ** 3) @ M3.T).reshape(-1)
    np.testing.assert_allclose(op.apply(ub), Mf, atol=1e-14)
    del one


def test_lowest_eigenvalue_three_pi_squared():
    """lambda_min(A, M) -> 3 pi^2, the first Dirichlet eigenvalue of the unit cube."""
    p, N = 2, 4
    m = Mesh(N=(N, N, N))
    op = SIPG(m, p)
    A = op.assemble()
    t = basis1d.tables(p)
    h = 1.0 / N
    Mloc = h * (t["S"].T * t["wq"]) @ t["S"]
    M = np.kron(np.eye(m.ncells), np.kron(Mloc, np.kron(Mloc, Mloc)))
    import scipy.linalg as sla
    lam = sla.eigh(0.5 * (A + A.T), M, eigvals_only=True, subset_by_index=[0, 0])[0]
    assert abs(lam - 3 * np.pi ** 2) < 2e-3 * 3 * np.pi ** 2


# ---------------------------------------------------------------- invariants
GEOMS = {
    "cartesian": dict(),
    "paper_affine": dict(L=(1.12, 0.24, 0.36, 0.24, 1.36, 0.48, 0.36, 0.48, 1.60),
                         lo=(-0.95, -0.9, -0.85), hi=(0.95, 0.89, 0.83)),
    "curved": dict(amp=0.05),                                                  # BASELINE C3 map
}


@pytest.mark.parametrize("geom", list(GEOMS))
@pytest.mark.parametrize("p", [1, 2, 3])
def test_symmetric_positive_definite_mirror(geom, p):
    m = Mesh(N=(2, 2, 2), **GEOMS[geom])
    A = SIPG(m, p).assemble()
    assert np.abs(A - A.T).max() <= 1e-13 * np.abs(A).max()
    assert np.linalg.eigvalsh(0.5 * (A + A.T))[0] > 0


@pytest.mark.parametrize("geom", list(GEOMS))
@pytest.mark.parametrize("p", [2, 3])
def test_periodic_constant_nullspace(geom, p):
    m = Mesh(N=(3, 2, 2), bc=("periodic",) * 3, **GEOMS[geom])
    op = SIPG(m, p)
    one = np.ones(m.ncells * (p + 1) ** 3)
    y = op.apply(one)
    assert np.abs(y).max() < 1e-12 * (p + 1) ** 2 * 3


@pytest.mark.parametrize("geom", ["paper_affine", "curved"])
@pytest.mark.parametrize("p", [2, 4])
def test_cross_basis_identity(geom, p):
    """Same space and quadrature: A_H = T3^T A_GL T3 cell-blockwise."""
    m = Mesh(N=(2, 2, 1), **GEOMS[geom])
    AH = SIPG(m, p).assemble()
    AG = SIPG(m, p, "gl").assemble()
    T = np.kron(np.eye(m.ncells), sm.T3(p))
    assert np.abs(AH - T.T @ AG @ T).max() <= 1e-12 * np.abs(AH).max()


def test_jacobian_matches_finite_differences():
    m = Mesh(N=(3, 4, 5), amp=0.05, L=(1.1, 0.2, 0.0, 0.1, 0.9, 0.3, 0.0, 0.2, 1.2))
    rng = np.random.default_rng(3)
    xi = rng.uniform(0.1, 0.9, (7, 3))
    cells = np.array([0, 17, 59])
    J = m.jacobian(cells, xi)
    eps = 1e-6
    for k in range(3):
        dx = np.zeros(3)
        dx[k] = eps
        fd = (m.position(cells, xi + dx) - m.position(cells, xi - dx)) / (2 * eps)
        np.testing.assert_allclose(J[..., :, k], fd, atol=1e-8)
    detJ = np.linalg.det(m.jacobian(np.arange(60), xi)) * 3 * 4 * 5 / (1.1 * 0.9 * 1.2 - 0.1 * 0.2 * 1.2 - 1.1 * 0.3 * 0.2 + 0.0)
    assert np.all(detJ > 0)


@pytest.mark.parametrize("p", [2, 3])
def test_ones_energy_equals_boundary_penalty_curved(p):
    """For u = 1 only the mirror penalty survives: 1'A1 = sum_boundary 2 sigma_F A_F, with
    A_F integrated here from |J e_t1 x J e_t2| (tangent cross product), not Nanson's formula,
    and sigma_F = (p+1)^2 A_F / V_K, V_K = sum_q w_q det J_q."""
    m = Mesh(N=(2, 2, 2), amp=0.05)
    op = SIPG(m, p)
    one = np.ones(m.ncells * (p + 1) ** 3)
    lhs = one @ op.apply(one)
    t = basis1d.tables(p)
    n = p + 1
    total = 0.0
    for c in range(m.ncells):
        V = op.volumes(np.array([c]))[0]
        cc = m.cell_coords(np.array([c]))[0]
        for d in range(3):
            for s in (0, 1):
                if (s == 0 and cc[d] != 0) or (s == 1 and cc[d] != m.N[d] - 1):
                    continue
                t1, t2 = [k for k in range(3) if k != d]
                pts = np.zeros((n * n, 3))
                a = np.arange(n * n)
                pts[:, t1], pts[:, t2], pts[:, d] = t["xq"][a % n], t["xq"][a // n], s
                w = t["wq"][a % n] * t["wq"][a // n]
                J = m.jacobian(np.array([c]), pts)[0]
                area = np.sum(np.linalg.norm(np.cross(J[:, :, t1], J[:, :, t2]), axis=-1) * w)
                total += 2 * (p + 1) ** 2 * area / V * area
    assert abs(lhs - total) < 1e-11 * total


def test_diagonal_matches_assembled():
    m = Mesh(N=(2, 2, 2), amp=0.05, bc=("dirichlet", "periodic", "dirichlet"))
    for basis in ("hermite", "gl"):
        op = SIPG(m, 2, basis)
        np.testing.assert_allclose(op.diagonal(), np.diag(op.assemble()), rtol=1e-14, atol=1e-13)


def test_gl_diagonal_cartesian_kronecker():
    """On Cartesian meshes diag(A_GL) = sum of Kronecker products of 1D diagonals (Eq. (14))."""
    N = (3, 2, 2)
    p = 3
    m = Mesh(N=N)
    d = SIPG(m, p, "gl").diagonal()
    K = kron_sum_3d(p, N, (0, 0, 0), (1, 1, 1), ("dirichlet",) * 3, "gl")
    np.testing.assert_allclose(d, np.diag(K), rtol=1e-13)
