"""dg_mesh_desc.user_penalty: the caller's sigma_F per face, in face
order 2d+s per owned cell, equal on the two sides of every face (PAPER.md:167-170 gives
the default (p+1)^2 A_F/V_K that this input replaces).  GPU parity of the matvec, both
inverse diagonals and the fused Chebyshev step with a random penalty field against the
oracle given the same field, on Cartesian, per-cell affine and curved meshes; the error
paths of the input (mismatched sides, negative / non-finite values)."""
import numpy as np
import pytest
import torch

from synthetic import MeshSpec, uniform_vector

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


def random_face_penalty(spec, rng, lo=0.8, hi=2.0):
    """(ncells, 6) array: one random sigma per face of the global mesh, copied to both cells
    of the face (periodic faces wrap), face order 2d+s; sigma = (p+1)^2 N_d/|box_d| times
    U(lo, hi), i.e. around the default penalty (well-conditioned, coercive operator)."""
    N = spec.n_cells
    p = spec.degree
    nc = N[0] * N[1] * N[2]
    out = np.empty((nc, 6))
    for d in range(3):
        # face planes 0..N_d-1 under periodic (plane N_d == plane 0), 0..N_d otherwise
        nplanes = N[d] if spec.bc[d] == "periodic" else N[d] + 1
        shape = [N[0], N[1], N[2]]
        shape[d] = nplanes
        base = (p + 1) ** 2 * N[d] / (spec.box_hi[d] - spec.box_lo[d])
        sig = base * rng.uniform(lo, hi, size=shape[::-1])   # [z][y][x] with plane index along d
        for c in range(nc):
            cc = [c % N[0], (c // N[0]) % N[1], c // (N[0] * N[1])]
            for s in (0, 1):
                pl = cc[d] + s
                if spec.bc[d] == "periodic":
                    pl %= N[d]
                idx = list(cc)
                idx[d] = pl
                out[c, 2 * d + s] = sig[idx[2], idx[1], idx[0]]
    return out


CASES = [
    ("cartesian", dict(n_cells=(4, 3, 3), box_hi=(1.0, 0.8, 1.2), bc=("periodic", "dirichlet", "periodic"))),
    ("paper_affine", dict(n_cells=(3, 2, 3), box_lo=(-0.95, -0.9, -0.85), box_hi=(0.95, 0.89, 0.83),
                          linear_map=PAPER_L, bc=("dirichlet", "periodic", "dirichlet"))),
    ("per_cell", dict(n_cells=(3, 2, 3), box_lo=(-0.95, -0.9, -0.85), box_hi=(0.95, 0.89, 0.83),
                      linear_map=PAPER_L, geometry="per_cell", bc=("dirichlet", "periodic", "dirichlet"))),
    ("curved", dict(n_cells=(3, 2, 3), deform_amp=0.05, geometry="per_qpoint",
                    bc=("dirichlet", "dirichlet", "periodic"))),
]


@pytest.mark.parametrize("case", [c[0] for c in CASES])
@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_user_penalty_parity(case, p):
    _needs_gpu()
    import paper_1907_08492_b200 as P
    from oracle import smoother as sm
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    spec = MeshSpec(degree=p, seed=1400 + p, **dict(CASES)[case])
    up = random_face_penalty(spec, np.random.default_rng(1400 + p))
    om = mesh_from_spec(spec)
    H = SIPG(om, p, "hermite", user_penalty=up)
    G = SIPG(om, p, "gl", user_penalty=up)
    m = P.mesh_from_spec(spec, user_penalty=up)
    u = uniform_vector(spec.n_dofs, spec.seed)
    ref = H.apply(u)
    assert _rel(m.apply_laplace(_dev(u)).cpu().numpy(), ref) <= TOL
    # the field matters: the default penalty gives a different operator
    assert _rel(SIPG(om, p).apply(u), ref) > 1e-3
    dgl = G.diagonal()
    assert _rel(m.inverse_diagonal("gl_jacobi").cpu().numpy(), 1 / dgl) <= TOL
    assert _rel(m.inverse_diagonal("point_jacobi").cpu().numpy(), 1 / H.diagonal()) <= TOL
    b = uniform_vector(spec.n_dofs, spec.seed + 7)
    lmax = 2.6
    ref_x = sm.chebyshev(H.apply, sm.GLJacobi(G), b, u, 2, lmax)
    x = _dev(u)
    m.chebyshev_smooth(_dev(b), x, lmax, degree=2)
    assert _rel(x.cpu().numpy(), ref_x) <= TOL


def test_user_penalty_uniform_equals_default_cartesian():
    """A user field equal to the default (p+1)^2/h_d on a Cartesian mesh reproduces the
    default operator (Kronecker kernel) through the general kernels."""
    _needs_gpu()
    import paper_1907_08492_b200 as P
    p = 3
    spec = MeshSpec(degree=p, n_cells=(4, 3, 2), box_hi=(1.0, 0.6, 1.0), seed=1500)
    h = [1.0 / 4, 0.6 / 3, 1.0 / 2]
    up = np.empty((spec.n_cells_total, 6))
    for d in range(3):
        up[:, 2 * d] = up[:, 2 * d + 1] = (p + 1) ** 2 / h[d]
    u = _dev(uniform_vector(spec.n_dofs, 1500))
    y0 = P.mesh_from_spec(spec).apply_laplace(u).cpu().numpy()
    y1 = P.mesh_from_spec(spec, user_penalty=up).apply_laplace(u).cpu().numpy()
    assert _rel(y1, y0) <= TOL


def test_user_penalty_errors():
    _needs_gpu()
    import paper_1907_08492_b200 as P
    spec = MeshSpec(degree=2, n_cells=(3, 2, 2), bc=("periodic", "dirichlet", "dirichlet"))
    up = random_face_penalty(spec, np.random.default_rng(0))
    bad = up.copy()
    bad[1, 0] *= 1.5                      # x-face between cells 0 and 1 differs on the two sides
    with pytest.raises(P.DgError, match="DG_ERR_PARAM.*differs"):
        P.mesh_from_spec(spec, user_penalty=bad)
    bad = up.copy()
    bad[0, 1] = bad[2, 0] = up[0, 1] * 2  # periodic wrap face: cell 2 (x=2) face 1 vs cell 0 face 0
    bad[0, 0] = up[0, 0] * 3
    with pytest.raises(P.DgError, match="DG_ERR_PARAM"):
        P.mesh_from_spec(spec, user_penalty=bad)
    bad = up.copy()
    bad[3, 4] = -1.0
    with pytest.raises(P.DgError, match="DG_ERR_PARAM.*negative"):
        P.mesh_from_spec(spec, user_penalty=bad)
    bad = up.copy()
    bad[5, 2] = np.nan
    with pytest.raises(P.DgError, match="DG_ERR_PARAM"):
        P.mesh_from_spec(spec, user_penalty=bad)
    with pytest.raises(ValueError, match="user_penalty"):
        P.mesh_from_spec(spec, user_penalty=up[:-1])
    # the Cartesian-only paths refuse a mesh with per-face penalties
    m = P.mesh_from_spec(spec, user_penalty=up)
    b = torch.zeros(spec.n_dofs, dtype=torch.float64, device="cuda")
    with pytest.raises(P.DgError, match="UNSUPPORTED"):
        m.chebyshev_smooth(b, b.clone(), 2.0, degree=1, inner="fdm")
    with pytest.raises(P.DgError, match="UNSUPPORTED"):
        m.apply_laplace_f32(b.float())


def test_misaligned_vector_rejected():
    """dg.h: vector pointers must be 16-byte aligned; a view at an odd element offset is
    refused (DG_ERR_PARAM from the library, ValueError from the binding) instead of
    faulting in a 128-bit access."""
    _needs_gpu()
    import ctypes
    import paper_1907_08492_b200 as P
    from paper_1907_08492_b200._lib import lib
    spec = MeshSpec(degree=3, n_cells=(2, 2, 2))
    m = P.mesh_from_spec(spec)
    buf = torch.zeros(spec.n_dofs + 1, dtype=torch.float64, device="cuda")
    y = torch.zeros(spec.n_dofs, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError, match="aligned"):
        m.apply_laplace(buf[1:], y)
    st = lib().dg_apply_laplace(m._h, ctypes.c_void_p(buf.data_ptr() + 8), ctypes.c_void_p(y.data_ptr()), 0,
                                ctypes.c_void_p(0))
    assert st == 1 and b"aligned" in lib().dg_last_error()
    # the context is still healthy
    m.apply_laplace(buf[:-1], y)
    torch.cuda.synchronize()
