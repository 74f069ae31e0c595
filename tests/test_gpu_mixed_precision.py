"""Single / mixed precision (the paper's smoothers and preconditioners
run in fp32): the fp32 basis change and CG in fp64 around an fp32
Chebyshev preconditioner (dg_pcg_mixed).

Tolerances.  fp32 basis change: the input is rounded to float once and the fp64 oracle is
applied to the rounded input, so the difference is the fp32 arithmetic alone: 3 even-odd
sweeps of about n/2 + 2 rounded operations each, unit roundoff 6e-8, |B| entries <= 2.3
and cond(B^{x3}) <= 12.5 (SURVEY.md §8(c) basis-change pins): relative L2 <= 3 (n/2+2)
6e-8 * 12.5 < 2e-5; measured values are far below, the test uses TOL32 = 2e-6 as the
other fp32 tests.  Mixed PCG: the fp32 preconditioner is a perturbation of size ~1e-7 of a
fixed SPD operator, which changes CG's iterates but not its fixed point: the solution must
reach the fp64 tolerance and agree with the dense solve like dg_pcg does."""
import numpy as np
import pytest
import torch

from synthetic import MeshSpec, uniform_vector

pytestmark = pytest.mark.gpu
TOL32 = 2e-6


def _needs_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("p", range(1, 9))
@pytest.mark.parametrize("op", ["T", "Tinv", "TT", "TinvT"])
def test_basis_change_f32(p, op):
    _needs_gpu()
    import paper_1907_08492_b200 as P
    from oracle import smoother as sm
    spec = MeshSpec(degree=p, n_cells=(5, 3, 2), seed=1600 + p)
    u32 = uniform_vector(spec.n_dofs, spec.seed).astype(np.float32)
    ref = sm.basis_change(p, u32.astype(np.float64), op)
    m = P.mesh_from_spec(spec)
    v = m.basis_change_f32(op, torch.from_numpy(u32).cuda()).cpu().numpy().astype(np.float64)
    assert _rel(v, ref) <= TOL32
    w = torch.from_numpy(u32).cuda()
    m.basis_change_f32(op, w, out=w)                      # in place
    assert _rel(w.cpu().numpy().astype(np.float64), ref) <= TOL32


@pytest.mark.parametrize("p,inner", [(3, "gl_jacobi"), (4, "fdm"), (5, "point_jacobi")])
def test_pcg_mixed_solves(p, inner):
    _needs_gpu()
    import paper_1907_08492_b200 as P
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    spec = MeshSpec(degree=p, n_cells=(3, 2, 3), bc=("dirichlet", "periodic", "dirichlet"), seed=1700 + p)
    A = SIPG(mesh_from_spec(spec), p).assemble()
    b = uniform_vector(spec.n_dofs, spec.seed)
    xs = np.linalg.solve(A, b)
    m = P.mesh_from_spec(spec)
    lmax = m.lanczos_lambda_max(inner if inner != "point_jacobi" else "point_jacobi", 15)
    bd = torch.from_numpy(b).cuda()
    x64 = torch.zeros_like(bd)
    it64, res64 = m.pcg(bd, x64, lmax, rel_tol=1e-11, max_iter=300, cheby_degree=3, inner=inner)
    xm = torch.zeros_like(bd)
    itm, resm = m.pcg_mixed(bd, xm, lmax, rel_tol=1e-11, max_iter=300, cheby_degree=3, inner=inner)
    assert resm <= 1e-11 and res64 <= 1e-11
    assert itm <= it64 + 3                       # fp32 preconditioning costs at most a few iterations
    assert _rel(xm.cpu().numpy(), xs) <= 1e-9
    assert _rel(x64.cpu().numpy(), xs) <= 1e-9


def test_pcg_mixed_unsupported_on_curved():
    _needs_gpu()
    import paper_1907_08492_b200 as P
    spec = MeshSpec(degree=3, n_cells=(2, 2, 2), deform_amp=0.05, geometry="per_qpoint")
    m = P.mesh_from_spec(spec)
    b = torch.ones(spec.n_dofs, dtype=torch.float64, device="cuda")
    with pytest.raises(P.DgError, match="UNSUPPORTED"):
        m.pcg_mixed(b, torch.zeros_like(b), 2.5)
