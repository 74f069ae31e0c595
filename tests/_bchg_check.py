"""Basis-change parity run in a subprocess by test_gpu_variants.py (the kernel-selection
environment variables are read once per process): every op at p = 1..8 against the oracle,
out of place and in place, fp64 (1e-12) and fp32, on meshes of 18, 105 and 1771 cells so that
tiles are ragged and (with DG_BCHGW_GRID=2) every warp streams many tiles through its slots.
Prints "OK"."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_08492_b200 as P  # noqa: E402
from oracle import smoother as sm  # noqa: E402
from synthetic import MeshSpec, uniform_vector  # noqa: E402

TOL, TOL32 = 1e-12, 2e-6


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def main():
    for p in range(1, 9):
        for nc in ((3, 2, 3), (7, 5, 3), (23, 11, 7)):
            spec = MeshSpec(degree=p, n_cells=nc, seed=900 + p)
            m = P.mesh_from_spec(spec)
            u = uniform_vector(spec.n_dofs, spec.seed)
            for op in (("T", "Tinv", "TT", "TinvT") if nc[0] != 23 else ("T", "TinvT")):
                ref = sm.basis_change(p, u, op)
                d = torch.from_numpy(u).cuda()
                e = rel(m.basis_change(op, d).cpu().numpy(), ref)
                assert e <= TOL, (p, nc, op, "out of place", e)
                m.basis_change(op, d, out=d)
                e = rel(d.cpu().numpy(), ref)
                assert e <= TOL, (p, nc, op, "in place", e)
                u32 = u.astype(np.float32)
                ref32 = sm.basis_change(p, u32.astype(np.float64), op)
                d32 = torch.from_numpy(u32).cuda()
                e = rel(m.basis_change_f32(op, d32).cpu().numpy().astype(np.float64), ref32)
                assert e <= TOL32, (p, nc, op, "f32", e)
                m.basis_change_f32(op, d32, out=d32)
                e = rel(d32.cpu().numpy().astype(np.float64), ref32)
                assert e <= TOL32, (p, nc, op, "f32 in place", e)
    print("OK", flush=True)


if __name__ == "__main__":
    main()
