"""Worker of test_gpu_nccl_multirank.py, launched by torch.distributed.run with one process per
GPU: the library's own NCCL data plane (dg_halo_exchange inside every operator pass, the
interior/boundary overlap on the comm stream, ncclAllReduce in dg_dot) against the single-rank
result computed on rank 0.  Checks: the slab-split matvec and the fused Chebyshev sweep equal
the single rank BIT FOR BIT (same per-cell arithmetic), Lanczos and PCG (dot products summed
across ranks by NCCL) agree to 1e-12 / 1e-9; periodic z with two ranks makes both peers of a
rank the same process.  Prints "OK" on rank 0."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_08492_b200 as P  # noqa: E402
from synthetic import MeshSpec, uniform_vector  # noqa: E402


def gather(local, total):
    """Concatenate the ranks' slab vectors (rank order = z order) on every rank."""
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, local.cpu().numpy())
    out = np.concatenate(parts)
    assert out.size == total
    return out


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count())
    dist.init_process_group("gloo")   # control plane only (unique id, gathers); data plane is NCCL
    cases = [
        (MeshSpec(degree=2, n_cells=(7, 3, 8), bc=("periodic", "dirichlet", "dirichlet"), seed=61), "gl_jacobi"),
        (MeshSpec(degree=3, n_cells=(5, 4, 8), bc=("dirichlet", "periodic", "periodic"), seed=62), "gl_jacobi"),
        (MeshSpec(degree=5, n_cells=(3, 3, 6), bc=("dirichlet", "dirichlet", "periodic"), seed=63), "point_jacobi"),
        (MeshSpec(degree=4, n_cells=(3, 2, 6), bc=("dirichlet", "periodic", "dirichlet"), seed=64), "fdm"),
        (MeshSpec(degree=3, n_cells=(2, 3, 6), deform_amp=0.05, geometry="per_qpoint", seed=65), "gl_jacobi"),
    ]
    for spec, inner in cases:
        obj = [P.get_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        m = P.mesh_from_spec(spec, rank=rank, nranks=world, nccl_unique_id=obj[0] if world > 1 else None)
        single = P.mesh_from_spec(spec)   # every rank: the whole mesh on its own GPU
        plane = spec.n_cells[0] * spec.n_cells[1] * spec.n ** 3
        sl = slice(m.z_begin * plane, m.z_end * plane)
        u = torch.from_numpy(uniform_vector(spec.n_dofs, spec.seed)).cuda()
        b = torch.from_numpy(uniform_vector(spec.n_dofs, spec.seed + 100)).cuda()
        tag = (spec.degree, spec.n_cells, spec.bc, inner)
        # matvec (halo exchange + overlap inside the call)
        y = gather(m.apply_laplace(u[sl].clone()), spec.n_dofs)
        assert np.array_equal(y, single.apply_laplace(u).cpu().numpy()), ("apply", tag)
        # fused Chebyshev sweep, one exchange per step
        lm = 2.5
        x = u[sl].clone()
        m.chebyshev_smooth(b[sl].clone(), x, lm, degree=4, inner=inner)
        xr = u.clone()
        single.chebyshev_smooth(b, xr, lm, degree=4, inner=inner)
        assert np.array_equal(gather(x, spec.n_dofs), xr.cpu().numpy()), ("chebyshev", tag)
        # dot (ncclAllReduce), Lanczos, PCG
        d = m.dot(u[sl].clone(), u[sl].clone())
        dr = single.dot(u, u)
        assert abs(d - dr) <= 1e-13 * abs(dr), ("dot", tag, d, dr)
        if spec.geometry == "constant" or inner == "gl_jacobi":
            e = m.lanczos_lambda_max(inner, 15)
            er = single.lanczos_lambda_max(inner, 15)
            assert abs(e - er) <= 1e-12 * er, ("lanczos", tag, e, er)
        xs = torch.zeros(m.n_local_dofs, dtype=torch.float64, device="cuda")
        it, rel = m.pcg(b[sl].clone(), xs, 2.6, rel_tol=1e-10, max_iter=200, cheby_degree=3, inner=inner)
        x1 = torch.zeros_like(b)
        it1, rel1 = single.pcg(b, x1, 2.6, rel_tol=1e-10, max_iter=200, cheby_degree=3, inner=inner)
        assert it == it1 and rel <= 1e-10, ("pcg", tag, it, it1, rel)
        xg = gather(xs, spec.n_dofs)
        x1 = x1.cpu().numpy()
        assert np.linalg.norm(xg - x1) <= 1e-9 * np.linalg.norm(x1), ("pcg x", tag)
        del m
        dist.barrier()
    if rank == 0:
        print("OK", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
