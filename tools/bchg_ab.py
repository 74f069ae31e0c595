"""A/B timing of the standalone basis change (row a12) on the C4 meshes; the kernel is picked
by DG_BCHG (1 = cell-staged k_bchg, 4 = z-first k_bchg4) in the environment of the process."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_08492_b200 as P  # noqa: E402
from synthetic import c4_spec  # noqa: E402

res = {}
for p in range(2, 9):
    spec = c4_spec(p)
    m = P.mesh_from_spec(spec)
    x = torch.rand(m.n_local_dofs, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        m.basis_change("TinvT", x, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    K = 20
    for _ in range(K):
        m.basis_change("TinvT", x, out=y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    res[p] = round(16 * m.n_local_dofs / (ms * 1e-3) / 1e9)
    del m, x, y
print(os.environ.get("DG_BCHG", "default"), res, flush=True)
