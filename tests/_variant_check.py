"""Parity checks run in a subprocess by test_gpu_variants.py, so that the kernel-selection
environment variables (read once per process by the library) take effect.  Checks the matvec,
the fused Chebyshev step (GL-Jacobi and point Jacobi) and the basis change against the oracle
on meshes whose rows span several blocks (ragged last block, periodic wrap).  Prints "OK"."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_08492_b200 as P  # noqa: E402
from oracle import smoother as sm  # noqa: E402
from oracle.geometry import mesh_from_spec  # noqa: E402
from oracle.sipg import SIPG  # noqa: E402
from synthetic import MeshSpec, uniform_vector  # noqa: E402

TOL = 1e-12


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def main(degrees, curved):
    for p in degrees:
        for nc, bcx in (((19, 3, 2), "periodic"), ((21, 2, 3), "dirichlet"), ((45, 2, 2), "periodic")):
            geoms = [("constant", 0.0)] + ([("per_qpoint", 0.03)] if curved else [])
            for geom, amp in geoms:
                spec = MeshSpec(degree=p, n_cells=nc, bc=(bcx, "periodic", "dirichlet"), geometry=geom,
                                deform_amp=amp, seed=700 + p)
                om = mesh_from_spec(spec)
                H = SIPG(om, p)
                m = P.mesh_from_spec(spec)
                u = uniform_vector(spec.n_dofs, spec.seed)
                e = rel(m.apply_laplace(dev(u)).cpu().numpy(), H.apply(u))
                assert e <= TOL, (p, nc, geom, "apply", e)
                if nc[0] == 45:   # rows of several blocks with a periodic wrap between blocks
                    continue
                b = uniform_vector(spec.n_dofs, 710 + p)
                cheb = p <= 5 and nc[0] == 19   # the oracle smoother setup is slow beyond that
                for inner, Pc in ((("gl_jacobi", sm.GLJacobi(SIPG(om, p, "gl"))),
                                   ("point_jacobi", sm.PointJacobi(H))) if cheb else ()):
                    ref = sm.chebyshev(H.apply, Pc, b, u, 2, 2.4)
                    x = dev(u)
                    m.chebyshev_smooth(dev(b), x, 2.4, degree=2, inner=inner)
                    e = rel(x.cpu().numpy(), ref)
                    assert e <= TOL, (p, nc, geom, inner, e)
                if geom == "constant":
                    for op in ("T", "TinvT"):
                        e = rel(m.basis_change(op, dev(u)).cpu().numpy(), sm.basis_change(p, u, op))
                        assert e <= TOL, (p, nc, "bchg", op, e)
    print("OK", flush=True)


if __name__ == "__main__":
    main([int(x) for x in sys.argv[1].split(",")], len(sys.argv) > 2 and sys.argv[2] == "curved")
