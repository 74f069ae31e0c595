"""Small driver for ncu captures: one C4 mesh of degree p, W warm-up rounds then one round of
the ops (matvec, basis change, degree-2 Chebyshev), all through the public binding.

    python tools/prof_driver.py P [ops=apply,bchg,cheby] [rounds=2]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1907_08492_b200 as P  # noqa: E402
from synthetic import CONFIGS, c4_spec  # noqa: E402

p = sys.argv[1]   # a C4 degree, or a BASELINE config name (C2, C3, C5)
ops = (sys.argv[2] if len(sys.argv) > 2 else "apply,bchg,cheby").split(",")
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 2
spec = CONFIGS[p] if p in CONFIGS else c4_spec(int(p))
m = P.mesh_from_spec(spec)
g = torch.Generator(device="cuda").manual_seed(1)
u = torch.rand(m.n_local_dofs, dtype=torch.float64, device="cuda", generator=g)
b = torch.rand_like(u)
y = torch.empty_like(u)
x = torch.zeros_like(u)
w2 = torch.empty(2 * u.numel(), dtype=torch.float64, device="cuda")
for _ in range(rounds):
    if "apply" in ops:
        m.apply_laplace(u, y)
    if "bchg" in ops:
        m.basis_change("T", u, y)
    if "cheby" in ops:
        m.chebyshev_smooth(b, x, 2.4, degree=2, work2=w2)
torch.cuda.synchronize()
print("ok", p, ops)
