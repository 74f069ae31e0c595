"""Basis-change kernels for compute-sanitizer (memcheck / racecheck): every degree p = 1..8 on a
mesh of 105 cells (ragged tiles), out of place and in place, fp64 and fp32; the kernel and mode
come from the environment (DG_BCHG, DG_BCHGW_MODE, DG_BCHGW_GRID=2 so warps reuse their slots)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_08492_b200 as P  # noqa: E402
from synthetic import MeshSpec, uniform_vector  # noqa: E402

for p in range(1, 9):
    spec = MeshSpec(degree=p, n_cells=(7, 5, 3), seed=p)
    m = P.mesh_from_spec(spec)
    u = torch.from_numpy(uniform_vector(spec.n_dofs, p)).cuda()
    m.basis_change("T", u)
    m.basis_change("TinvT", u, out=u)
    w = u.float()
    m.basis_change_f32("Tinv", w)
    m.basis_change_f32("TT", w, out=w)
torch.cuda.synchronize()
print("ok")
