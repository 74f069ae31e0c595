"""GPU parity of the general quadrature kernel (k_quad: the paper's formulation,
Eqs. (3)-(5)) against the CPU oracle: constant affine geometry,
per-cell J^-1, per-quadrature-point curved geometry (BASELINE C3), diagonals and
the fused Chebyshev step on non-Cartesian meshes.  Relative L2 <= 1e-12."""
import numpy as np
import pytest
import torch

from synthetic import CONFIGS, MeshSpec, uniform_vector

pytestmark = pytest.mark.gpu
TOL = 1e-12
PAPER_L = (1.12, 0.24, 0.36, 0.24, 1.36, 0.48, 0.36, 0.48, 1.60)


def _needs_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _oracle(spec, inv_jac=None):
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    om = mesh_from_spec(spec)
    if inv_jac is not None:
        om.inv_jac = inv_jac
    return SIPG(om, spec.degree, spec.basis, spec.penalty_factor)


def _gpu(spec, **kw):
    import paper_1907_08492_b200 as P
    return P.mesh_from_spec(spec, **kw)


@pytest.mark.parametrize("p", range(1, 9))
@pytest.mark.parametrize("basis", ["hermite", "gl"])
def test_quadrature_flag_on_cartesian(p, basis):
    """The general kernel on a Cartesian mesh (DG_APPLY_QUADRATURE) equals the oracle."""
    _needs_gpu()
    import paper_1907_08492_b200 as P
    spec = MeshSpec(degree=p, n_cells=(3, 2, 3), basis=basis, box_lo=(0, -0.5, 0.25), box_hi=(1.5, 0.5, 1.0),
                    bc=("dirichlet", "periodic", "dirichlet"), seed=70 + p)
    u = uniform_vector(spec.n_dofs, spec.seed)
    ref = _oracle(spec).apply(u)
    y = _gpu(spec).apply_laplace(_dev(u), flags=P.APPLY_QUADRATURE).cpu().numpy()
    assert _rel(y, ref) <= TOL


@pytest.mark.parametrize("p", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("geometry", ["constant", "per_cell", "per_qpoint"])
def test_paper_affine_geometry(p, geometry):
    """The paper's §5 affine brick in all three storage modes."""
    _needs_gpu()
    spec = MeshSpec(degree=p, n_cells=(2, 3, 2), box_lo=(-0.95, -0.9, -0.85), box_hi=(0.95, 0.89, 0.83),
                    linear_map=PAPER_L, geometry=geometry, bc=("dirichlet", "dirichlet", "periodic"),
                    seed=80 + p)
    u = uniform_vector(spec.n_dofs, spec.seed)
    ref = _oracle(spec).apply(u)
    y = _gpu(spec).apply_laplace(_dev(u)).cpu().numpy()
    assert _rel(y, ref) <= TOL


@pytest.mark.parametrize("p", [2, 4, 7])
def test_per_cell_user_inverse_jacobians(p):
    """DG_GEOM_PER_CELL with a user array of per-cell J^-1 (varying cell to cell)."""
    _needs_gpu()
    spec = MeshSpec(degree=p, n_cells=(3, 2, 2), geometry="per_cell", bc=("periodic", "dirichlet", "dirichlet"),
                    seed=90 + p)
    rng = np.random.default_rng(p)
    nc = spec.n_cells_total
    base = np.linalg.inv(np.diag([1 / 3, 1 / 2, 1 / 2]))
    ji = np.array([base + 0.3 * rng.uniform(-1, 1, (3, 3)) for _ in range(nc)])
    u = uniform_vector(spec.n_dofs, spec.seed)
    ref = _oracle(spec, inv_jac=ji).apply(u)
    y = _gpu(spec, user_inv_jac=ji.reshape(nc, 9)).apply_laplace(_dev(u)).cpu().numpy()
    assert _rel(y, ref) <= TOL


@pytest.mark.parametrize("p", range(1, 9))
@pytest.mark.parametrize("bc", ["dirichlet", "periodic"])
def test_curved_per_qpoint(p, bc):
    """BASELINE C3 map (amp 0.05) on small meshes, per-quadrature-point geometry."""
    _needs_gpu()
    spec = MeshSpec(degree=p, n_cells=(3, 2, 3), deform_amp=0.05, geometry="per_qpoint", bc=(bc,) * 3,
                    seed=110 + p)
    u = uniform_vector(spec.n_dofs, spec.seed)
    ref = _oracle(spec).apply(u)
    y = _gpu(spec).apply_laplace(_dev(u)).cpu().numpy()
    assert _rel(y, ref) <= TOL


def test_curved_gl_basis():
    _needs_gpu()
    spec = MeshSpec(degree=4, n_cells=(2, 3, 2), basis="gl", deform_amp=0.05, geometry="per_qpoint", seed=5)
    u = uniform_vector(spec.n_dofs, spec.seed)
    ref = _oracle(spec).apply(u)
    assert _rel(_gpu(spec).apply_laplace(_dev(u)).cpu().numpy(), ref) <= TOL


def test_c3_full_size_sampled():
    """BASELINE C3: p=5, 48^3 curved cells, per-q-point geometry, seed 2 (23.9M DoF);
    200 sampled cells (corners included) against the oracle."""
    _needs_gpu()
    spec = CONFIGS["C3"]
    u = uniform_vector(spec.n_dofs, spec.seed)
    y = _gpu(spec).apply_laplace(_dev(u)).cpu().numpy().reshape(spec.n_cells_total, -1)
    N = spec.n_cells
    rng = np.random.default_rng(3)
    cells = np.unique(np.concatenate([[0, N[0] - 1, N[0] * N[1] - 1, spec.n_cells_total - 1],
                                      rng.choice(spec.n_cells_total, 200, replace=False)]))
    ref = _oracle(spec).apply(u, cells=cells).reshape(len(cells), -1)
    assert np.abs(y[cells] - ref).max() <= TOL * np.abs(ref).max()


@pytest.mark.parametrize("geometry,amp", [("per_qpoint", 0.05), ("constant", 0.0), ("per_cell", 0.0)])
@pytest.mark.parametrize("p", [2, 5])
def test_general_diagonals(geometry, amp, p):
    _needs_gpu()
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    L = PAPER_L if amp == 0.0 else (1, 0, 0, 0, 1, 0, 0, 0, 1)
    spec = MeshSpec(degree=p, n_cells=(2, 3, 2), linear_map=L, deform_amp=amp, geometry=geometry,
                    bc=("dirichlet", "periodic", "dirichlet"))
    om = mesh_from_spec(spec)
    m = _gpu(spec)
    assert _rel(m.inverse_diagonal("gl_jacobi").cpu().numpy(), 1 / SIPG(om, p, "gl").diagonal()) <= TOL
    assert _rel(m.inverse_diagonal("point_jacobi").cpu().numpy(), 1 / SIPG(om, p).diagonal()) <= TOL


@pytest.mark.parametrize("inner", ["gl_jacobi", "point_jacobi"])
@pytest.mark.parametrize("p", [3, 6])
def test_chebyshev_curved(inner, p):
    _needs_gpu()
    from oracle import smoother as sm
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    spec = MeshSpec(degree=p, n_cells=(2, 2, 3), deform_amp=0.05, geometry="per_qpoint", seed=120 + p)
    om = mesh_from_spec(spec)
    H = SIPG(om, p)
    P = sm.GLJacobi(SIPG(om, p, "gl")) if inner == "gl_jacobi" else sm.PointJacobi(H)
    b = uniform_vector(spec.n_dofs, 700 + p)
    x0 = uniform_vector(spec.n_dofs, 800 + p)
    ref = sm.chebyshev(H.apply, P, b, x0, 5, 2.5)
    x = _dev(x0)
    _gpu(spec).chebyshev_smooth(_dev(b), x, 2.5, degree=5, inner=inner)
    assert _rel(x.cpu().numpy(), ref) <= TOL


def test_numeric_error_on_inverted_map():
    _needs_gpu()
    import paper_1907_08492_b200 as P
    with pytest.raises(P.DgError, match="DG_ERR_NUMERIC"):
        P.Mesh(degree=2, n_cells=(2, 2, 2), deform_amp=2.0, geometry="per_qpoint")
