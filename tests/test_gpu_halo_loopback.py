"""Multi-rank path on ONE GPU with the external halo transport ("loopback backend",
SURVEY.md §4 item 4): G virtual z-slab ranks, each its own mesh handle; the halo
planes are packed by the library (dg_halo_pack), moved between the virtual ranks by
device copies, installed with dg_halo_set, and every slab is applied with
DG_APPLY_HALO_READY.  The concatenated result must equal the single-rank result
bit for bit (same per-cell arithmetic), for the Kronecker and the quadrature kernels."""
import numpy as np
import pytest
import torch

from synthetic import MeshSpec, uniform_vector

pytestmark = pytest.mark.gpu


def _run(spec, G, flags=0):
    import paper_1907_08492_b200 as P
    u = torch.from_numpy(uniform_vector(spec.n_dofs, spec.seed)).cuda()
    ref = P.mesh_from_spec(spec).apply_laplace(u, flags=flags)
    meshes = [P.mesh_from_spec(spec, rank=r, nranks=G) for r in range(G)]
    plane = spec.n_cells[0] * spec.n_cells[1] * spec.n ** 3
    slabs = [u[m.z_begin * plane:m.z_end * plane].contiguous() for m in meshes]
    packs = [m.halo_pack(s) for m, s in zip(meshes, slabs)]
    outs = []
    for r, m in enumerate(meshes):
        h = m.query_halo()
        recv_lo = packs[h["lo_peer"]][1] if h["lo_peer"] >= 0 else None   # lower peer's top planes
        recv_hi = packs[h["hi_peer"]][0] if h["hi_peer"] >= 0 else None   # upper peer's bottom planes
        m.halo_set(recv_lo, recv_hi)
        outs.append(m.apply_laplace(slabs[r], flags=flags | P.APPLY_HALO_READY))
    return torch.cat(outs), ref


@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("bc", ["dirichlet", "periodic"])
@pytest.mark.parametrize("p,basis", [(2, "hermite"), (5, "hermite"), (3, "gl")])
def test_loopback_kron(G, bc, p, basis):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    spec = MeshSpec(degree=p, n_cells=(3, 2, 5), basis=basis, bc=("dirichlet", "periodic", bc), seed=31)
    y, ref = _run(spec, G)
    assert torch.equal(y, ref)


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("bc", ["dirichlet", "periodic"])
def test_loopback_quadrature_curved(G, bc):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    spec = MeshSpec(degree=4, n_cells=(2, 3, 4), deform_amp=0.05, geometry="per_qpoint",
                    bc=("dirichlet", "dirichlet", bc), seed=32)
    y, ref = _run(spec, G)
    assert torch.equal(y, ref)


def test_external_transport_requires_halo_ready():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1907_08492_b200 as P
    spec = MeshSpec(degree=3, n_cells=(2, 2, 4))
    m = P.mesh_from_spec(spec, rank=0, nranks=2)
    u = torch.zeros(m.n_local_dofs, dtype=torch.float64, device="cuda")
    with pytest.raises(P.DgError, match="UNSUPPORTED"):
        m.apply_laplace(u)


def test_c5_slab_sampled():
    """BASELINE C5 shape (p=5, 128^3) split in 8 virtual slabs; the slab results of the
    first two ranks (including the interface) equal the single-rank result."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1907_08492_b200 as P
    spec = MeshSpec(degree=5, n_cells=(128, 128, 128), seed=4)
    g = torch.Generator(device="cuda").manual_seed(4)
    u = torch.rand(spec.n_dofs, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    plane = 128 * 128 * 216
    single = P.mesh_from_spec(spec)
    ref = single.apply_laplace(u)[: 32 * plane].clone()
    del single
    G = 8
    ms = [P.mesh_from_spec(spec, rank=r, nranks=G) for r in range(3)]
    slabs = [u[m.z_begin * plane:m.z_end * plane] for m in ms]
    packs = [m.halo_pack(s) for m, s in zip(ms, slabs)]
    outs = []
    for r in range(2):
        m = ms[r]
        h = m.query_halo()
        m.halo_set(packs[h["lo_peer"]][1] if h["lo_peer"] >= 0 else None, packs[r + 1][0])
        outs.append(m.apply_laplace(slabs[r], flags=P.APPLY_HALO_READY))
    assert torch.equal(torch.cat(outs), ref)
