"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck):
k_kron4 (apply, Chebyshev GL/PJ/FDM, fp32), k_quad3 and k_quad (apply, Chebyshev), basis
change, the solver layer.  Ragged meshes, mixed boundary conditions."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_08492_b200 as P  # noqa: E402
from synthetic import MeshSpec, uniform_vector  # noqa: E402

dev = torch.device("cuda", 0)


def v(n, s, dt=torch.float64):
    return torch.from_numpy(uniform_vector(n, s)).to(dev, dt)


for p in (2, 3, 5, 8):
    spec = MeshSpec(degree=p, n_cells=(3, 2, 4), bc=("dirichlet", "periodic", "dirichlet"), seed=p)
    m = P.mesh_from_spec(spec)
    n = m.n_local_dofs
    u, b = v(n, 1), v(n, 2)
    m.apply_laplace(u)
    m.basis_change("T", u)
    for inner in ("gl_jacobi", "point_jacobi", "fdm"):
        x = torch.zeros(n, dtype=torch.float64, device=dev)
        m.chebyshev_smooth(b, x, 2.0, degree=3, inner=inner)
        m.apply_preconditioner(b, inner=inner)
    m.apply_laplace_f32(u.float())
    x32 = torch.zeros(n, dtype=torch.float32, device=dev)
    m.chebyshev_smooth_f32(b.float(), x32, 2.0, degree=3, inner="fdm")
    lm = m.lanczos_lambda_max("gl_jacobi", 5)
    m.pcg(b, torch.zeros(n, dtype=torch.float64, device=dev), lm, max_iter=3, cheby_degree=2)
    for geom, amp in (("per_qpoint", 0.05), ("per_cell", 0.0), ("constant", 0.0)):
        spec2 = MeshSpec(degree=p, n_cells=(3, 2, 3), deform_amp=amp, geometry=geom, seed=p)
        m2 = P.mesh_from_spec(spec2)
        u2 = v(m2.n_local_dofs, 3)
        m2.apply_laplace(u2)
        x2 = torch.zeros_like(u2)
        m2.chebyshev_smooth(v(m2.n_local_dofs, 4), x2, 2.0, degree=2)
torch.cuda.synchronize()
print("sanitize run ok")
