"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck):
k_kron4 (apply, Chebyshev GL/PJ/FDM, fp32), k_kron6 (the i-plane kernel at n = 3..6, forced
on for apply and Chebyshev with DG_K6=255 in the environment), k_quad3 and k_quad (apply,
Chebyshev), basis change (fp64 and fp32), the solver layer (PCG, mixed PCG), user
penalties.  Ragged meshes, mixed boundary conditions."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_08492_b200 as P  # noqa: E402
from synthetic import MeshSpec, uniform_vector  # noqa: E402

dev = torch.device("cuda", 0)


def v(n, s, dt=torch.float64):
    return torch.from_numpy(uniform_vector(n, s)).to(dev, dt)


for p in (2, 3, 4, 5, 8):
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
    m.pcg_mixed(b, torch.zeros(n, dtype=torch.float64, device=dev), lm, max_iter=3, cheby_degree=2)
    m.basis_change_f32("TinvT", u.float())
    # rows of several blocks with a periodic wrap (k_kron6 virtual halo cells, k_kron4 jobs)
    spec3 = MeshSpec(degree=p, n_cells=(45, 2, 2), bc=("periodic", "dirichlet", "periodic"), seed=p)
    m3 = P.mesh_from_spec(spec3)
    u3 = v(m3.n_local_dofs, 5)
    m3.apply_laplace(u3)
    m3.chebyshev_smooth(v(m3.n_local_dofs, 6), torch.zeros_like(u3), 2.0, degree=2)
    import numpy as np
    pen = np.full((spec.n_cells_total, 6), 30.0 * (p + 1) ** 2)
    m4 = P.mesh_from_spec(spec, user_penalty=pen)
    m4.apply_laplace(u)
    m4.chebyshev_smooth(b, torch.zeros_like(u), 2.0, degree=2)
    for geom, amp in (("per_qpoint", 0.05), ("per_cell", 0.0), ("constant", 0.0)):
        spec2 = MeshSpec(degree=p, n_cells=(3, 2, 3), deform_amp=amp, geometry=geom, seed=p)
        m2 = P.mesh_from_spec(spec2)
        u2 = v(m2.n_local_dofs, 3)
        m2.apply_laplace(u2)
        x2 = torch.zeros_like(u2)
        m2.chebyshev_smooth(v(m2.n_local_dofs, 4), x2, 2.0, degree=2)
torch.cuda.synchronize()
print("sanitize run ok")
