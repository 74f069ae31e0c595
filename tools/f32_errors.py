"""Print the measured fp32 relative L2 errors of the matvec and Chebyshev (GPU vs fp64
oracle on rounded inputs) for DESIGN.md."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1907_08492_b200 as P
from oracle import smoother as sm
from oracle.geometry import mesh_from_spec
from oracle.sipg import SIPG
from synthetic import MeshSpec, uniform_vector

for p in range(2, 9):
    spec = MeshSpec(degree=p, n_cells=(3, 2, 4), box_hi=(1.0, 0.8, 1.3),
                    bc=("dirichlet", "periodic", "dirichlet"), seed=110 + p)
    u32 = uniform_vector(spec.n_dofs, spec.seed).astype(np.float32)
    om = mesh_from_spec(spec)
    H = SIPG(om, p)
    ref = H.apply(u32.astype(np.float64))
    m = P.mesh_from_spec(spec)
    y = m.apply_laplace_f32(torch.from_numpy(u32).cuda()).cpu().numpy().astype(np.float64)
    e1 = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    b32 = uniform_vector(spec.n_dofs, 130 + p).astype(np.float32)
    x32 = uniform_vector(spec.n_dofs, 140 + p).astype(np.float32)
    refx = sm.chebyshev(H.apply, sm.GLJacobi(SIPG(om, p, "gl")), b32.astype(np.float64), x32.astype(np.float64), 5, 2.0)
    x = torch.from_numpy(x32).cuda()
    m.chebyshev_smooth_f32(torch.from_numpy(b32).cuda(), x, 2.0, degree=5)
    e2 = np.linalg.norm(x.cpu().numpy() - refx) / np.linalg.norm(refx)
    print(f"p={p} matvec_f32 rel L2 {e1:.2e}  chebyshev_f32 (degree 5) rel L2 {e2:.2e}", flush=True)
