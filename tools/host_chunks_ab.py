"""e2e matvec through dg_apply_laplace_host (pinned host vectors) on the C4 meshes for several
z-chunk counts (DG_HOST_CHUNKS is read per call)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_08492_b200 as P  # noqa: E402
from synthetic import c4_spec  # noqa: E402

for p in (2, 5, 8):
    m = P.mesh_from_spec(c4_spec(p))
    n = m.n_local_dofs
    uh = torch.rand(n, dtype=torch.float64).pin_memory()
    yh = torch.empty(n, dtype=torch.float64).pin_memory()
    s = torch.cuda.current_stream()
    res = {}
    for ch in (8, 16, 32, 64, 8, 32):
        os.environ["DG_HOST_CHUNKS"] = str(ch)
        m.apply_laplace_host(uh, yh)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(3):
            m.apply_laplace_host(uh, yh)
        e1.record(s)
        torch.cuda.synchronize()
        res.setdefault(ch, []).append(round(3 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2))
    print(p, res, flush=True)
    del m, uh, yh
