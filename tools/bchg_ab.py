"""A/B timing of the standalone basis change (row a12) on the C4 meshes; the kernel is picked
by DG_BCHG (1 = cell-staged k_bchg, 4 = z-first k_bchg4) in the environment of the process."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_08492_b200 as P  # noqa: E402
from synthetic import c4_spec  # noqa: E402

f32 = "--f32" in sys.argv          # fp32 basis change (dg_basis_change_f32), 8 B/DoF
res = {}
for p in range(2, 9):
    spec = c4_spec(p)
    m = P.mesh_from_spec(spec)
    x = torch.rand(m.n_local_dofs, dtype=torch.float32 if f32 else torch.float64, device="cuda")
    y = torch.empty_like(x)
    bc = m.basis_change_f32 if f32 else m.basis_change
    for _ in range(3):
        bc("TinvT", x, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    K = 20
    for _ in range(K):
        bc("TinvT", x, out=y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    res[p] = round((8 if f32 else 16) * m.n_local_dofs / (ms * 1e-3) / 1e9)
    del m, x, y
print(os.environ.get("DG_BCHG", "default"), "f32" if f32 else "f64", res, flush=True)
