"""GPU parity of the fused Chebyshev step (Eqs. (11)-(12))
at every degree p = 1..8 on multi-block meshes, one and two steps at the FULL C4 / C3
sizes on sampled cells, and the penalty factor of dg_mesh_setup (sigma = pf (p+1)^2 A_F/V_K,
PAPER.md:167-170) on the Cartesian, per-cell and curved kernels.

Tolerance: relative L2 <= 1e-12 in fp64 (BASELINE.json north_star), max-abs per element
<= 1e-12 max|oracle| on the sampled checks.  Inputs are seeded uniform[-1,1) vectors.

Cost control (test side only, no arithmetic of the method here): on a Cartesian mesh of
equal cells the diagonal of a cell depends only on which of its faces are mirror
boundaries or self-periodic, because every cell has the same Jacobian J = L diag(h)
bit for bit.  `_diag_by_class` therefore asks the oracle for one representative cell
per face class and copies its diagonal to the other cells of the class.
"""
import numpy as np
import pytest
import torch

from synthetic import CONFIGS, MeshSpec, c4_spec, uniform_vector

pytestmark = pytest.mark.gpu
TOL = 1e-12
PAPER_L = (1.12, 0.24, 0.36, 0.24, 1.36, 0.48, 0.36, 0.48, 1.60)

# cells per block of the z-first Cartesian kernel for n = p+1 (csrc/k_kron4.cu K4C<n>::CPB);
# the meshes below take Nx = CPB + a ragged remainder so each x-row spans >= 2 blocks
CPB = {1: 8, 2: 32, 3: 30, 4: 16, 5: 8, 6: 10, 7: 4, 8: 3}


def _needs_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _gpu(spec, **kw):
    import paper_1907_08492_b200 as P
    return P.mesh_from_spec(spec, **kw)


def _face_class(om, cells):
    cc = om.cell_coords(cells)
    key = []
    for d in range(3):
        N = om.N[d]
        key.append((cc[:, d] == 0).astype(int) + 2 * (cc[:, d] == N - 1) + 4 * (N == 1))
    return key[0] + 8 * key[1] + 64 * key[2]


def _diag_by_class(op, cells):
    """diag(A) rows of `cells` for a Cartesian (uniform-cell) mesh, one oracle call per class."""
    om = op.mesh
    cells = np.asarray(cells)
    cls = _face_class(om, cells)
    n3 = op.n ** 3
    out = np.empty((len(cells), n3))
    for c in np.unique(cls):
        rep = cells[cls == c][0]
        out[cls == c] = op.diagonal(cells=np.array([rep]))
    return out.reshape(-1)


def _pinv_cells(p, inner, dinv_cells, r_cells):
    """P^{-1} restricted to whole cells (block-diagonal preconditioners)."""
    from oracle import smoother as sm
    if inner == "point_jacobi":
        return r_cells * dinv_cells
    z = sm.basis_change(p, r_cells, "TinvT") * dinv_cells
    return sm.basis_change(p, z, "Tinv")


_DINV_CACHE = {}


@pytest.mark.parametrize("p", range(1, 9))
@pytest.mark.parametrize("inner", ["gl_jacobi", "point_jacobi"])
@pytest.mark.parametrize("degree", [1, 2, 5])
def test_chebyshev_every_degree_multiblock(p, inner, degree):
    """Eq. (11) with the inner GL-Jacobi (Eq. (12)) or point-Jacobi preconditioner at every
    p on rows of >= 2 blocks with a ragged last block, >= 3 planes, mixed boundaries."""
    _needs_gpu()
    from oracle import smoother as sm
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    Nx = CPB[p] + max(1, CPB[p] // 2 + 1)
    spec = MeshSpec(degree=p, n_cells=(Nx, 2, 3), box_hi=(1.0, 0.7, 1.1),
                    bc=("periodic", "dirichlet", "dirichlet"), seed=900 + p)
    om = mesh_from_spec(spec)
    H = SIPG(om, p)
    key = (p, inner)
    if key not in _DINV_CACHE:       # the three sweep degrees share the mesh and its diagonal
        dop = SIPG(om, p, "gl") if inner == "gl_jacobi" else H
        _DINV_CACHE[key] = 1.0 / _diag_by_class(dop, np.arange(om.ncells))
    dinv = _DINV_CACHE[key]
    P = (lambda r: _pinv_cells(p, inner, dinv, r))
    b = uniform_vector(spec.n_dofs, 910 + p)
    x0 = uniform_vector(spec.n_dofs, 920 + p)
    lmax = 2.4
    ref = sm.chebyshev(H.apply, P, b, x0, degree, lmax)
    m = _gpu(spec)
    x = _dev(x0)
    m.chebyshev_smooth(_dev(b), x, lmax, degree=degree, inner=inner)
    assert _rel(x.cpu().numpy(), ref) <= TOL


def _neighbours(om, cells):
    """cells and their face neighbours (periodic wrap / clipped at mirror faces)."""
    cc = om.cell_coords(np.asarray(cells))
    out = [np.asarray(cells)]
    for d in range(3):
        for s in (-1, 1):
            c2 = cc.copy()
            c2[:, d] += s
            if om.bc[d] == "periodic":
                c2[:, d] %= om.N[d]
            else:
                c2[:, d] = np.clip(c2[:, d], 0, om.N[d] - 1)
            out.append(om.cell_id(c2))
    return np.unique(np.concatenate(out))


def _sample(N, k, rng):
    Nx, Ny, Nz = N
    corners = [0, Nx - 1, Nx * Ny - 1, Nx * Ny * Nz - 1, Nx * Ny * (Nz - 1), Nx * Ny * (Nz // 2) + Nx // 2]
    return np.unique(np.concatenate([corners, rng.choice(Nx * Ny * Nz, size=k, replace=False)]))


def _two_steps_sampled(spec, m, inner, lmax, cartesian, ncells_sample, seed):
    """x_1 and x_2 of Eq. (11) (degree-2 sweep) on sampled cells S of a full-size mesh:
    x_1 = x_0 + P^{-1}(b - A x_0)/c on S1 = S + neighbours(S), then
    x_2 = x_1 + rho_2 rho_1 (x_1 - x_0) + (2 rho_2/delta) P^{-1}(b - A x_1) on S, which needs
    x_1 only on S1 (A is a nearest-neighbour operator)."""
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    p = spec.degree
    n3 = spec.n ** 3
    g = torch.Generator(device="cuda").manual_seed(seed)
    x0d = torch.rand(spec.n_dofs, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    bd = torch.rand(spec.n_dofs, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    x0 = x0d.cpu().numpy()
    b = bd.cpu().numpy()
    om = mesh_from_spec(spec)
    H = SIPG(om, p, spec.basis, spec.penalty_factor)
    dop = SIPG(om, p, "gl", spec.penalty_factor) if inner == "gl_jacobi" else H
    S = _sample(spec.n_cells, ncells_sample, np.random.default_rng(seed))
    S1 = _neighbours(om, S)
    diag = (lambda c: _diag_by_class(dop, c)) if cartesian else (lambda c: dop.diagonal(cells=c))
    dinv1 = 1.0 / diag(S1)
    alpha, beta = 0.06 * lmax, 1.2 * lmax
    c, delta = 0.5 * (beta + alpha), 0.5 * (beta - alpha)
    r0 = b.reshape(-1, n3)[S1].reshape(-1) - H.apply(x0, cells=S1)
    x1_S1 = x0.reshape(-1, n3)[S1].reshape(-1) + (1.0 / c) * _pinv_cells(p, inner, dinv1, r0)
    # GPU, degree 1 (the first-step kernel, u_{j-1} not read)
    x = x0d.clone()
    m.chebyshev_smooth(bd, x, lmax, degree=1, inner=inner)
    x1g = x.view(-1, n3)[torch.from_numpy(S1).cuda()].cpu().numpy().reshape(-1)
    del x
    # x_2 on S from x_1 on S1
    x1 = x0.copy()
    x1.reshape(-1, n3)[S1] = x1_S1.reshape(-1, n3)
    sig1 = c / delta
    rho1 = 1.0 / sig1
    rho2 = 1.0 / (2.0 * sig1 - rho1)
    pos = np.searchsorted(S1, S)
    dinvS = dinv1.reshape(-1, n3)[pos].reshape(-1)
    x1S = x1.reshape(-1, n3)[S].reshape(-1)
    x0S = x0.reshape(-1, n3)[S].reshape(-1)
    rS = b.reshape(-1, n3)[S].reshape(-1) - H.apply(x1, cells=S)
    x2S = x1S + rho2 * rho1 * (x1S - x0S) + (2.0 * rho2 / delta) * _pinv_cells(p, inner, dinvS, rS)
    x = x0d.clone()
    m.chebyshev_smooth(bd, x, lmax, degree=2, inner=inner)
    x2g = x.view(-1, n3)[torch.from_numpy(S).cuda()].cpu().numpy().reshape(-1)
    return (x1g, x1_S1), (x2g, x2S)


@pytest.mark.parametrize("p", range(2, 9))
def test_c4_full_size_chebyshev_sampled(p):
    """C4 sweep meshes (108-113M DoF) in the bench launch configuration: the first and the
    second fused Chebyshev step (GL-Jacobi) against the oracle on sampled cells."""
    _needs_gpu()
    spec = c4_spec(p)
    m = _gpu(spec)
    (g1, r1), (g2, r2) = _two_steps_sampled(spec, m, "gl_jacobi", 2.5, True, 24, 1000 + p)
    assert np.abs(g1 - r1).max() <= TOL * np.abs(r1).max()
    assert _rel(g1, r1) <= TOL
    assert np.abs(g2 - r2).max() <= TOL * np.abs(r2).max()
    assert _rel(g2, r2) <= TOL


@pytest.mark.parametrize("inner", ["gl_jacobi", "point_jacobi"])
def test_c3_full_size_chebyshev_sampled(inner):
    """BASELINE C3 (p=5, 48^3 curved, per-q-point geometry, 23.9M DoF): first and second
    fused Chebyshev step of the general kernel on sampled cells."""
    _needs_gpu()
    spec = CONFIGS["C3"]
    m = _gpu(spec)
    (g1, r1), (g2, r2) = _two_steps_sampled(spec, m, inner, 2.5, False, 12, 1100)
    assert _rel(g1, r1) <= TOL
    assert _rel(g2, r2) <= TOL


def test_c5_full_size_chebyshev_sampled():
    """BASELINE C5 on one GPU (p=5, 128^3 cells, 453M DoF): the int64 offsets of the
    fused step, first and second step on sampled cells."""
    _needs_gpu()
    spec = CONFIGS["C5"]
    m = _gpu(spec)
    (g1, r1), (g2, r2) = _two_steps_sampled(spec, m, "gl_jacobi", 2.4, True, 8, 1200)
    assert _rel(g1, r1) <= TOL
    assert _rel(g2, r2) <= TOL


# ---------------------------------------------------------------- penalty factor
PF_CASES = [
    ("cartesian", dict(n_cells=(5, 3, 3), box_hi=(1.0, 0.8, 1.2))),
    ("per_cell", dict(n_cells=(3, 2, 3), box_lo=(-0.95, -0.9, -0.85), box_hi=(0.95, 0.89, 0.83),
                      linear_map=PAPER_L, geometry="per_cell")),
    ("curved", dict(n_cells=(3, 2, 3), deform_amp=0.05, geometry="per_qpoint")),
]


@pytest.mark.parametrize("pf", [0.5, 2.5])
@pytest.mark.parametrize("case", [c[0] for c in PF_CASES])
@pytest.mark.parametrize("p", [2, 3, 5])
def test_penalty_factor(pf, case, p):
    """sigma_F = pf (p+1)^2 A_F/V_K (dg_mesh_desc.penalty_factor): matvec,
    both inverse diagonals and a degree-2 Chebyshev sweep against the oracle with the same pf."""
    _needs_gpu()
    from oracle import smoother as sm
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    kw = dict(PF_CASES)[case]
    spec = MeshSpec(degree=p, bc=("dirichlet", "periodic", "dirichlet"), penalty_factor=pf,
                    seed=1300 + p, **kw)
    om = mesh_from_spec(spec)
    H = SIPG(om, p, "hermite", pf)
    G = SIPG(om, p, "gl", pf)
    u = uniform_vector(spec.n_dofs, spec.seed)
    m = _gpu(spec)
    assert _rel(m.apply_laplace(_dev(u)).cpu().numpy(), H.apply(u)) <= TOL
    dgl = G.diagonal()
    assert _rel(m.inverse_diagonal("gl_jacobi").cpu().numpy(), 1 / dgl) <= TOL
    assert _rel(m.inverse_diagonal("point_jacobi").cpu().numpy(), 1 / H.diagonal()) <= TOL
    b = uniform_vector(spec.n_dofs, 1310 + p)
    P = (lambda r: _pinv_cells(p, "gl_jacobi", 1 / dgl, r))
    ref = sm.chebyshev(H.apply, P, b, u, 2, 2.6)
    x = _dev(u)
    m.chebyshev_smooth(_dev(b), x, 2.6, degree=2)
    assert _rel(x.cpu().numpy(), ref) <= TOL
    # pf changes the operator: the pf = 1 result must differ by far more than the tolerance
    y1 = _gpu(spec.with_(penalty_factor=1.0)).apply_laplace(_dev(u)).cpu().numpy()
    assert _rel(y1, H.apply(u)) > 1e-3
