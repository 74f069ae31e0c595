"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerance: relative L2 <= 1e-12 in fp64 (BASELINE.json north_star), per
element |gpu - oracle| <= 1e-12 * max|oracle| on the sampled checks.
Inputs are seeded uniform[-1,1) vectors from synthetic/ (same bytes both sides).
"""
import numpy as np
import pytest
import torch

from synthetic import CONFIGS, MeshSpec, c4_spec, uniform_vector

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _needs_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _gpu_mesh(spec, **kw):
    import paper_1907_08492_b200 as P
    return P.mesh_from_spec(spec, **kw)


def _oracle(spec):
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    return SIPG(mesh_from_spec(spec), spec.degree, spec.basis, spec.penalty_factor)


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


SMALL = []
for p in range(1, 9):
    SMALL.append(MeshSpec(degree=p, n_cells=(3, 2, 4), box_lo=(0.0, -0.5, 0.25), box_hi=(1.5, 0.5, 1.0),
                          seed=100 + p))
    SMALL.append(MeshSpec(degree=p, n_cells=(5, 3, 2), bc=("periodic", "dirichlet", "periodic"),
                          seed=200 + p))
    SMALL.append(MeshSpec(degree=p, n_cells=(2, 3, 3), basis="gl", bc=("dirichlet", "periodic", "dirichlet"),
                          seed=300 + p))


@pytest.mark.parametrize("spec", SMALL, ids=lambda s: f"p{s.degree}-{s.basis}-{s.n_cells}-{s.bc[0][0]}{s.bc[1][0]}{s.bc[2][0]}")
def test_apply_small(spec):
    _needs_gpu()
    u = uniform_vector(spec.n_dofs, spec.seed)
    ref = _oracle(spec).apply(u)
    m = _gpu_mesh(spec)
    y = m.apply_laplace(_dev(u)).cpu().numpy()
    assert _rel(y, ref) <= TOL
    assert np.abs(y - ref).max() <= TOL * np.abs(ref).max()


def test_apply_c1_exact_config():
    """BASELINE C1: p=3, 4^3 cells, mirror Dirichlet, seed 0, 4096 DoF."""
    _needs_gpu()
    spec = CONFIGS["C1"]
    assert spec.n_dofs == 4096
    u = uniform_vector(spec.n_dofs, spec.seed)
    ref = _oracle(spec).apply(u)
    y = _gpu_mesh(spec).apply_laplace(_dev(u)).cpu().numpy()
    assert _rel(y, ref) <= TOL


def test_single_cell_and_periodic_self_neighbour():
    _needs_gpu()
    for bc in (("dirichlet",) * 3, ("periodic",) * 3, ("periodic", "dirichlet", "periodic")):
        for p in (2, 5):
            spec = MeshSpec(degree=p, n_cells=(1, 1, 1), bc=bc, seed=7)
            u = uniform_vector(spec.n_dofs, 7)
            ref = _oracle(spec).apply(u)
            y = _gpu_mesh(spec).apply_laplace(_dev(u)).cpu().numpy()
            assert _rel(y, ref) <= TOL, (bc, p)


@pytest.mark.parametrize("p", [2, 3, 5, 8])
def test_hermite_access_only_two_layers(p):
    """an interior cell reads its (p+1)^3 values plus 2 layers per
    face of each neighbour.  Poison every other neighbour coefficient with NaN:
    the cell's result must stay finite and bit-identical."""
    _needs_gpu()
    n = p + 1
    spec = MeshSpec(degree=p, n_cells=(3, 3, 3), seed=5)
    u = uniform_vector(spec.n_dofs, 5)
    m = _gpu_mesh(spec)
    y0 = m.apply_laplace(_dev(u)).cpu().numpy().reshape(27, n, n, n)
    U = u.reshape(3, 3, 3, n, n, n).copy()       # [cz,cy,cx,k,j,i]
    c = (1, 1, 1)
    poisoned = U.copy()
    for d in range(3):
        for s in (-1, 1):
            nb = list(c)
            nb[2 - d] += s
            cell = poisoned[tuple(nb)]
            keep = np.zeros((n, n, n), bool)
            layers = [n - 2, n - 1] if s < 0 else [0, 1]
            idx = [slice(None)] * 3
            idx[2 - d] = layers
            keep[tuple(idx)] = True
            cell[~keep] = np.nan
    y1 = m.apply_laplace(_dev(poisoned.reshape(-1))).cpu().numpy().reshape(27, n, n, n)
    centre = 13
    assert np.all(np.isfinite(y1[centre]))
    assert np.array_equal(y1[centre], y0[centre])


def test_gl_basis_reads_full_neighbours():
    """Nodal GL: the same poisoning must reach the centre cell."""
    _needs_gpu()
    p, n = 3, 4
    spec = MeshSpec(degree=p, n_cells=(3, 3, 3), basis="gl", seed=5)
    u = uniform_vector(spec.n_dofs, 5).reshape(3, 3, 3, n, n, n)
    u[1, 1, 0, :, :, 0] = np.nan          # x- neighbour, layer farthest from the face
    y = _gpu_mesh(spec).apply_laplace(_dev(u.reshape(-1))).cpu().numpy().reshape(27, -1)
    assert not np.all(np.isfinite(y[13]))


@pytest.mark.parametrize("p", range(1, 9))
@pytest.mark.parametrize("op", ["T", "Tinv", "TT", "TinvT"])
def test_basis_change(p, op):
    _needs_gpu()
    from oracle import smoother as sm
    spec = MeshSpec(degree=p, n_cells=(3, 2, 3), seed=40 + p)
    u = uniform_vector(spec.n_dofs, spec.seed)
    ref = sm.basis_change(p, u, op)
    m = _gpu_mesh(spec)
    v = m.basis_change(op, _dev(u)).cpu().numpy()
    assert _rel(v, ref) <= TOL
    w = _dev(u)
    m.basis_change(op, w, out=w)                   # in place
    assert _rel(w.cpu().numpy(), ref) <= TOL


@pytest.mark.parametrize("p", [2, 3, 5, 6, 8])
def test_basis_change_many_blocks(p):
    """z-first k_bchg4 over several blocks with a ragged last block (7*5*3 = 105 cells)."""
    _needs_gpu()
    from oracle import smoother as sm
    spec = MeshSpec(degree=p, n_cells=(7, 5, 3), seed=60 + p)
    u = uniform_vector(spec.n_dofs, spec.seed)
    m = _gpu_mesh(spec)
    for op in ("T", "TinvT"):
        ref = sm.basis_change(p, u, op)
        assert _rel(m.basis_change(op, _dev(u)).cpu().numpy(), ref) <= TOL


@pytest.mark.parametrize("p", [1, 2, 4, 7])
@pytest.mark.parametrize("basis", ["hermite", "gl"])
def test_inverse_diagonal(p, basis):
    _needs_gpu()
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    spec = MeshSpec(degree=p, n_cells=(3, 1, 2), basis=basis, bc=("dirichlet", "periodic", "dirichlet"))
    om = mesh_from_spec(spec)
    m = _gpu_mesh(spec)
    ref_gl = 1.0 / SIPG(om, p, "gl").diagonal()
    ref_pj = 1.0 / SIPG(om, p, basis).diagonal()
    assert _rel(m.inverse_diagonal("gl_jacobi").cpu().numpy(), ref_gl) <= TOL
    assert _rel(m.inverse_diagonal("point_jacobi").cpu().numpy(), ref_pj) <= TOL


@pytest.mark.parametrize("p", [2, 3, 5, 8])
@pytest.mark.parametrize("inner", ["gl_jacobi", "point_jacobi"])
@pytest.mark.parametrize("degree", [1, 2, 5])
def test_chebyshev(p, inner, degree):
    _needs_gpu()
    from oracle import smoother as sm
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    spec = MeshSpec(degree=p, n_cells=(3, 2, 2), bc=("dirichlet", "periodic", "dirichlet"), seed=60 + p)
    om = mesh_from_spec(spec)
    H = SIPG(om, p)
    P = sm.GLJacobi(SIPG(om, p, "gl")) if inner == "gl_jacobi" else sm.PointJacobi(H)
    b = uniform_vector(spec.n_dofs, 500 + p)
    x0 = uniform_vector(spec.n_dofs, 600 + p)
    lmax = 2.6
    ref = sm.chebyshev(H.apply, P, b, x0, degree, lmax)
    m = _gpu_mesh(spec)
    x = _dev(x0)
    m.chebyshev_smooth(_dev(b), x, lmax, degree=degree, inner=inner)
    assert _rel(x.cpu().numpy(), ref) <= TOL


@pytest.mark.parametrize("p", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("degree", [1, 3])
def test_chebyshev_fdm(p, degree):
    """Chebyshev around the FDM block-Jacobi inner preconditioner (Eqs. (13)-(15),
    PAPER.md:2117-2165) against oracle/fdm.py on an anisotropic, ragged mesh with
    mixed boundary conditions (interior-element matrices on every cell)."""
    _needs_gpu()
    from oracle import fdm
    from oracle import smoother as sm
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    spec = MeshSpec(degree=p, n_cells=(3, 2, 4), box_hi=(1.0, 0.8, 1.3),
                    bc=("dirichlet", "periodic", "dirichlet"), seed=70 + p)
    om = mesh_from_spec(spec)
    H = SIPG(om, p)
    P = fdm.FDM(p, (1.0 / 3, 0.8 / 2, 1.3 / 4))
    b = uniform_vector(spec.n_dofs, 700 + p)
    x0 = uniform_vector(spec.n_dofs, 800 + p)
    lmax = 1.7
    ref = sm.chebyshev(H.apply, P, b, x0, degree, lmax)
    m = _gpu_mesh(spec)
    x = _dev(x0)
    m.chebyshev_smooth(_dev(b), x, lmax, degree=degree, inner="fdm")
    assert _rel(x.cpu().numpy(), ref) <= TOL


def test_fdm_unsupported_on_curved_mesh():
    _needs_gpu()
    spec = MeshSpec(degree=3, n_cells=(2, 2, 2), deform_amp=0.05, geometry="per_qpoint", seed=1)
    m = _gpu_mesh(spec)
    b = _dev(uniform_vector(spec.n_dofs, 1))
    x = torch.zeros_like(b)
    with pytest.raises(Exception, match="FDM"):
        m.chebyshev_smooth(b, x, 2.0, degree=1, inner="fdm")


def _sample_cells(N, k, rng):
    Nx, Ny, Nz = N
    corners = [0, Nx - 1, Nx * Ny - 1, Nx * Ny * Nz - 1, Nx * Ny * (Nz - 1)]
    rest = rng.choice(Nx * Ny * Nz, size=k, replace=False)
    return np.unique(np.concatenate([corners, rest]))


@pytest.mark.parametrize("name", ["C2", "C2_GL"])
def test_c2_full_size_sampled(name):
    """BASELINE C2 (p=4, 32^3, 4.1M DoF, seed 1) in the bench launch configuration;
    the oracle computes 200 sampled cells (corners included) one by one."""
    _needs_gpu()
    spec = CONFIGS[name]
    u = uniform_vector(spec.n_dofs, spec.seed)
    y = _gpu_mesh(spec).apply_laplace(_dev(u)).cpu().numpy().reshape(spec.n_cells_total, -1)
    cells = _sample_cells(spec.n_cells, 200, np.random.default_rng(11))
    ref = _oracle(spec).apply(u, cells=cells).reshape(len(cells), -1)
    assert np.abs(y[cells] - ref).max() <= TOL * np.abs(ref).max()
    assert _rel(y[cells].ravel(), ref.ravel()) <= TOL


@pytest.mark.parametrize("p", range(2, 9))
def test_c4_full_size_sampled(p):
    """C4 sweep meshes (108-113M DoF) at full size: sampled-cell parity of the matvec
    and of one fused Chebyshev step (sampled via linearity: x_1 = x_0 + P^{-1}(b-Ax_0)/c)."""
    _needs_gpu()
    spec = c4_spec(p)
    n3 = spec.n ** 3
    g = torch.Generator(device="cuda").manual_seed(spec.seed)
    u = torch.rand(spec.n_dofs, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    m = _gpu_mesh(spec)
    y = m.apply_laplace(u)
    cells = _sample_cells(spec.n_cells, 40, np.random.default_rng(p))
    uh = u.cpu().numpy()
    yh = y.view(-1, n3)[torch.from_numpy(cells).cuda()].cpu().numpy()
    del y
    ref = _oracle(spec).apply(uh, cells=cells).reshape(len(cells), -1)
    assert np.abs(yh - ref).max() <= TOL * np.abs(ref).max()


# ---------------------------------------------------------------- solver layer (NEXT#4)
def _small_mesh(p=3, seed=80):
    return MeshSpec(degree=p, n_cells=(3, 2, 3), bc=("dirichlet", "periodic", "dirichlet"), seed=seed)


def test_gpu_dot_matches_numpy():
    _needs_gpu()
    spec = c4_spec(2)
    m = _gpu_mesh(spec)
    a = uniform_vector(m.n_local_dofs, 1)
    b = uniform_vector(m.n_local_dofs, 2)
    ref = float(np.dot(a, b))
    assert abs(m.dot(_dev(a), _dev(b)) - ref) <= 1e-12 * np.sqrt(np.dot(a, a) * np.dot(b, b))


@pytest.mark.parametrize("p", [2, 3, 5, 8])
@pytest.mark.parametrize("inner", ["gl_jacobi", "point_jacobi", "fdm"])
def test_gpu_apply_preconditioner(p, inner):
    _needs_gpu()
    from oracle import fdm
    from oracle import smoother as sm
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    spec = _small_mesh(p)
    om = mesh_from_spec(spec)
    if inner == "gl_jacobi":
        P = sm.GLJacobi(SIPG(om, p, "gl"))
    elif inner == "point_jacobi":
        P = sm.PointJacobi(SIPG(om, p))
    else:
        P = fdm.FDM(p, (1 / 3, 1 / 2, 1 / 3))
    r = uniform_vector(spec.n_dofs, 90 + p)
    m = _gpu_mesh(spec)
    z = m.apply_preconditioner(_dev(r), inner=inner).cpu().numpy()
    assert _rel(z, P(r)) <= TOL


@pytest.mark.parametrize("p,inner", [(3, "gl_jacobi"), (5, "gl_jacobi"), (4, "fdm"), (2, "point_jacobi")])
def test_gpu_lanczos_matches_oracle(p, inner):
    _needs_gpu()
    from oracle import fdm
    from oracle import smoother as sm
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    spec = _small_mesh(p)
    om = mesh_from_spec(spec)
    H = SIPG(om, p)
    P = {"gl_jacobi": lambda: sm.GLJacobi(SIPG(om, p, "gl")), "point_jacobi": lambda: sm.PointJacobi(H),
         "fdm": lambda: fdm.FDM(p, (1 / 3, 1 / 2, 1 / 3))}[inner]()
    ref = sm.lanczos_lambda_max(H.apply, P, spec.n_dofs, iters=15)
    m = _gpu_mesh(spec)
    assert abs(m.lanczos_lambda_max(inner=inner, iters=15) - ref) <= 1e-10 * ref


def test_gpu_lanczos_c1_sanity_value():
    """lambda_max(P^-1 A_H) for C1 (p=3, 4^3) is 2.592367.  A Lanczos Ritz
    value approaches lambda_max from below; 15 steps land within a few per cent."""
    _needs_gpu()
    m = _gpu_mesh(CONFIGS["C1"])
    est = m.lanczos_lambda_max("gl_jacobi", 15)
    assert 0.97 * 2.592367 <= est <= 2.592367 * (1 + 1e-9)


@pytest.mark.parametrize("inner,k", [("gl_jacobi", 3), ("fdm", 4)])
def test_gpu_pcg_iterates_match_oracle(inner, k):
    _needs_gpu()
    from oracle import fdm
    from oracle import smoother as sm
    from oracle import solver
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    p = 3
    spec = _small_mesh(p)
    om = mesh_from_spec(spec)
    H = SIPG(om, p)
    P = sm.GLJacobi(SIPG(om, p, "gl")) if inner == "gl_jacobi" else fdm.FDM(p, (1 / 3, 1 / 2, 1 / 3))
    lmax = 2.5
    M = lambda r: sm.chebyshev(H.apply, P, r, np.zeros_like(r), 3, lmax)   # noqa: E731
    b = uniform_vector(spec.n_dofs, 91)
    x0 = uniform_vector(spec.n_dofs, 92)
    xr, itr, resr = solver.pcg(H.apply, M, b, x0, rel_tol=0.0, max_iter=k)
    m = _gpu_mesh(spec)
    x = _dev(x0)
    it, res = m.pcg(_dev(b), x, lmax, rel_tol=0.0, max_iter=k, cheby_degree=3, inner=inner)
    assert it == itr == k
    assert _rel(x.cpu().numpy(), xr) <= 1e-10
    assert abs(res - resr) <= 1e-8 * resr


def test_gpu_pcg_solves():
    _needs_gpu()
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    spec = MeshSpec(degree=3, n_cells=(2, 2, 3), seed=5)
    A = SIPG(mesh_from_spec(spec), 3).assemble()
    b = uniform_vector(spec.n_dofs, 9)
    xs = np.linalg.solve(A, b)
    m = _gpu_mesh(spec)
    lmax = m.lanczos_lambda_max("gl_jacobi", 15)
    x = torch.zeros(spec.n_dofs, dtype=torch.float64, device="cuda")
    it, res = m.pcg(_dev(b), x, lmax, rel_tol=1e-11, max_iter=200, cheby_degree=3)
    assert res <= 1e-11 and it < 60
    assert _rel(x.cpu().numpy(), xs) <= 1e-9


# ---------------------------------------------------------------- fp32 path (NEXT#3)
# Tolerance: inputs are rounded to float once and the oracle is applied to
# the rounded input in fp64, so the difference is the fp32 arithmetic alone: ~50 rounded
# operations per output (7 even-odd sweeps + couplings) at unit roundoff 6e-8, amplified by
# the cancellation of the Laplacian of a random vector (|A||u| / |Au| ~ 3-10): <= 1e-5.
TOL32 = 2e-6   # bound 1e-5 (above); measured <= 1.9e-7 (profiles/r1_f32_errors.txt)


@pytest.mark.parametrize("p", [2, 3, 4, 5, 6, 7, 8])
def test_matvec_f32(p):
    _needs_gpu()
    spec = MeshSpec(degree=p, n_cells=(3, 2, 4), box_hi=(1.0, 0.8, 1.3),
                    bc=("dirichlet", "periodic", "dirichlet"), seed=110 + p)
    u32 = uniform_vector(spec.n_dofs, spec.seed).astype(np.float32)
    ref = _oracle(spec).apply(u32.astype(np.float64))
    m = _gpu_mesh(spec)
    y = m.apply_laplace_f32(torch.from_numpy(u32).cuda()).cpu().numpy().astype(np.float64)
    assert _rel(y, ref) <= TOL32


@pytest.mark.parametrize("p", [3, 5, 8])
@pytest.mark.parametrize("inner", ["gl_jacobi", "fdm", "point_jacobi"])
def test_chebyshev_f32(p, inner):
    _needs_gpu()
    from oracle import fdm
    from oracle import smoother as sm
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    spec = MeshSpec(degree=p, n_cells=(3, 2, 4), box_hi=(1.0, 0.8, 1.3),
                    bc=("dirichlet", "periodic", "dirichlet"), seed=120 + p)
    om = mesh_from_spec(spec)
    H = SIPG(om, p)
    P = {"gl_jacobi": lambda: sm.GLJacobi(SIPG(om, p, "gl")), "point_jacobi": lambda: sm.PointJacobi(H),
         "fdm": lambda: fdm.FDM(p, (1.0 / 3, 0.8 / 2, 1.3 / 4))}[inner]()
    b32 = uniform_vector(spec.n_dofs, 130 + p).astype(np.float32)
    x32 = uniform_vector(spec.n_dofs, 140 + p).astype(np.float32)
    lmax = 2.0
    ref = sm.chebyshev(H.apply, P, b32.astype(np.float64), x32.astype(np.float64), 3, lmax)
    m = _gpu_mesh(spec)
    x = torch.from_numpy(x32).cuda()
    m.chebyshev_smooth_f32(torch.from_numpy(b32).cuda(), x, lmax, degree=3, inner=inner)
    assert _rel(x.cpu().numpy().astype(np.float64), ref) <= TOL32


def test_f32_unsupported_on_curved_mesh():
    _needs_gpu()
    spec = MeshSpec(degree=3, n_cells=(2, 2, 2), deform_amp=0.05, geometry="per_qpoint", seed=1)
    m = _gpu_mesh(spec)
    u = torch.zeros(spec.n_dofs, dtype=torch.float32, device="cuda")
    with pytest.raises(Exception, match="fp32"):
        m.apply_laplace_f32(u)


@pytest.mark.parametrize("p", [2, 3, 5, 8])
@pytest.mark.parametrize("nc,bcx", [((11, 2, 2), "periodic"), ((13, 2, 3), "dirichlet"), ((33, 1, 2), "periodic")])
def test_rows_longer_than_a_block(p, nc, bcx):
    """Row-aligned blocks (k_kron4 / k_quad3): rows of several blocks with a ragged last
    block, the x-neighbours of the block-edge cells from halo jobs (periodic wrap across
    blocks), for the Cartesian and the curved per-q-point paths and the Chebyshev step."""
    _needs_gpu()
    from oracle import smoother as sm
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    for geom, amp in (("constant", 0.0), ("per_qpoint", 0.03)):
        spec = MeshSpec(degree=p, n_cells=nc, bc=(bcx, "periodic", "dirichlet"), geometry=geom,
                        deform_amp=amp, seed=150 + p)
        u = uniform_vector(spec.n_dofs, spec.seed)
        om = mesh_from_spec(spec)
        H = SIPG(om, p)
        m = _gpu_mesh(spec)
        assert _rel(m.apply_laplace(_dev(u)).cpu().numpy(), H.apply(u)) <= TOL, geom
        if geom == "constant":   # fp32 path on the same block structure
            u32 = u.astype(np.float32)
            y32 = m.apply_laplace_f32(torch.from_numpy(u32).cuda()).cpu().numpy().astype(np.float64)
            assert _rel(y32, H.apply(u32.astype(np.float64))) <= TOL32
        if p in (3, 5):
            b = uniform_vector(spec.n_dofs, 160 + p)
            ref = sm.chebyshev(H.apply, sm.GLJacobi(SIPG(om, p, "gl")), b, u, 2, 2.4)
            x = _dev(u)
            m.chebyshev_smooth(_dev(b), x, 2.4, degree=2)
            assert _rel(x.cpu().numpy(), ref) <= TOL, geom


@pytest.mark.parametrize("spec", [
    MeshSpec(degree=5, n_cells=(7, 5, 11), seed=170),                                         # chunked
    MeshSpec(degree=3, n_cells=(4, 3, 9), bc=("periodic", "dirichlet", "periodic"), seed=171),  # z-wrap
    MeshSpec(degree=4, n_cells=(3, 3, 8), deform_amp=0.04, geometry="per_qpoint", seed=172),   # k_quad3
    MeshSpec(degree=2, n_cells=(3, 2, 3), seed=173),                                          # < 4 planes
], ids=["chunked", "zwrap", "curved", "few-planes"])
def test_apply_host_buffers(spec):
    """dg_apply_laplace_host (HOST vectors, copies overlapped with the kernels) equals the
    device-vector matvec bit for bit; pinned and pageable host memory."""
    _needs_gpu()
    u = uniform_vector(spec.n_dofs, spec.seed)
    m = _gpu_mesh(spec)
    yd = m.apply_laplace(_dev(u)).cpu().numpy()
    for pinned in (True, False):
        uh = torch.from_numpy(u).pin_memory() if pinned else torch.from_numpy(u.copy())
        yh = m.apply_laplace_host(uh)
        torch.cuda.synchronize()
        assert np.array_equal(yh.numpy(), yd), pinned
    assert _rel(yd, _oracle(spec).apply(u)) <= TOL


@pytest.mark.parametrize("nc,bc", [((32, 2, 3), ("periodic", "dirichlet", "dirichlet")),
                                   ((64, 2, 2), ("dirichlet", "periodic", "periodic"))])
@pytest.mark.parametrize("basis", ["hermite", "gl"])
def test_k3c_full_tiles(nc, bc, basis):
    """k_kron3c's full-tile specialisation (rows a multiple of 32 cells, aligned vectors, no
    slab halo: the launcher picks the FAST kernel) for the matvec and the fused Chebyshev step
    with every inner preconditioner, against the oracle."""
    _needs_gpu()
    from oracle import fdm
    from oracle import smoother as sm
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    p = 2
    spec = MeshSpec(degree=p, n_cells=nc, bc=bc, basis=basis, seed=170)
    u = uniform_vector(spec.n_dofs, spec.seed)
    om = mesh_from_spec(spec)
    H = SIPG(om, p, basis)
    m = _gpu_mesh(spec)
    assert _rel(m.apply_laplace(_dev(u)).cpu().numpy(), H.apply(u)) <= TOL
    if basis != "hermite":
        return
    b = uniform_vector(spec.n_dofs, 171)
    h = tuple(1.0 / c for c in nc)
    for inner, Pc in (("gl_jacobi", sm.GLJacobi(SIPG(om, p, "gl"))), ("point_jacobi", sm.PointJacobi(H)),
                      ("fdm", fdm.FDM(p, h))):
        ref = sm.chebyshev(H.apply, Pc, b, u, 3, 2.4)
        x = _dev(u)
        m.chebyshev_smooth(_dev(b), x, 2.4, degree=3, inner=inner)
        assert _rel(x.cpu().numpy(), ref) <= TOL, inner
