"""The whole multi-slab layer on ONE GPU through the caller transport (dg_set_transport):
G virtual z-slab ranks, one host thread and one CUDA stream each, exchange the packed halo
planes inside every operator pass (the fused Chebyshev sweep: one halo per step,
PAPER.md:931-936) and sum the dot products of Lanczos and PCG on the host.  Nothing on
the GPU waits for another rank: the callbacks synchronise on the host (threading.Barrier)
and copy planes with dg_halo_set.

Checks: the Chebyshev sweep of every inner preconditioner equals the single-rank sweep
BIT FOR BIT (same per-cell arithmetic); Lanczos and PCG, whose dot products are summed
slab by slab, agree with the single rank to 1e-12 and with the oracle."""
import threading

import numpy as np
import pytest
import torch

from synthetic import MeshSpec, uniform_vector

pytestmark = pytest.mark.gpu


def _needs_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


class Loopback:
    """Host-side transport among G virtual ranks living in threads of this process."""

    def __init__(self, meshes):
        self.meshes = meshes
        self.G = len(meshes)
        self.bar = threading.Barrier(self.G, timeout=120)
        self.sends = [None] * self.G
        self.vals = [0.0] * self.G
        self.calls = 0

    def install(self, r):
        m = self.meshes[r]
        h = m.query_halo()
        lo, hi = h["lo_peer"], h["hi_peer"]

        def halo(slo, shi, rlo, rhi, count, stream):
            torch.cuda.current_stream().synchronize()   # the pack kernel of this rank is done
            self.sends[r] = (slo, shi)
            self.bar.wait()
            # lower peer's top planes -> recv_lo, upper peer's bottom planes -> recv_hi
            src_lo = self.sends[lo][1] if lo >= 0 else None
            src_hi = self.sends[hi][0] if hi >= 0 else None
            m.halo_set_raw(src_lo, src_hi)
            torch.cuda.current_stream().synchronize()
            self.bar.wait()                              # peers may overwrite their send planes
            if r == 0:
                self.calls += 1

        def allreduce(x):
            self.vals[r] = x
            self.bar.wait()
            s = 0.0
            for v in self.vals:                          # rank order: identical on every rank
                s += v
            self.bar.wait()
            return s

        m.set_transport(halo, allreduce)

    def run(self, fn):
        """fn(r) on every virtual rank concurrently (each on its own stream); returns results."""
        out = [None] * self.G
        err = []

        def body(r):
            try:
                with torch.cuda.stream(torch.cuda.Stream()):
                    out[r] = fn(r)
                    torch.cuda.current_stream().synchronize()
            except Exception as e:                      # noqa: BLE001
                err.append(e)
                self.bar.abort()

        ts = [threading.Thread(target=body, args=(r,)) for r in range(self.G)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if err:
            raise err[0]
        return out


def _setup(spec, G):
    import paper_1907_08492_b200 as P
    meshes = [P.mesh_from_spec(spec, rank=r, nranks=G) for r in range(G)]
    lb = Loopback(meshes)
    for r in range(G):
        lb.install(r)
    plane = spec.n_cells[0] * spec.n_cells[1] * spec.n ** 3
    sl = [slice(m.z_begin * plane, m.z_end * plane) for m in meshes]
    return P, meshes, lb, sl


@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("bcz", ["dirichlet", "periodic"])
@pytest.mark.parametrize("p,inner", [(2, "gl_jacobi"), (5, "gl_jacobi"), (3, "point_jacobi"), (4, "fdm")])
def test_chebyshev_sweep_slabs_bitwise(G, bcz, p, inner):
    _needs_gpu()
    spec = MeshSpec(degree=p, n_cells=(3, 2, 8), bc=("dirichlet", "periodic", bcz), seed=41)
    b = torch.from_numpy(uniform_vector(spec.n_dofs, 41)).cuda()
    x0 = torch.from_numpy(uniform_vector(spec.n_dofs, 42)).cuda()
    P, meshes, lb, sl = _setup(spec, G)
    ref = x0.clone()
    P.mesh_from_spec(spec).chebyshev_smooth(b, ref, 2.4, degree=4, inner=inner)
    xs = [x0[s].clone() for s in sl]
    bs = [b[s].clone() for s in sl]
    lb.run(lambda r: meshes[r].chebyshev_smooth(bs[r], xs[r], 2.4, degree=4, inner=inner))
    assert lb.calls == 4                                 # one exchange per Chebyshev step
    assert torch.equal(torch.cat(xs), ref)


@pytest.mark.parametrize("G", [2, 3])
def test_chebyshev_sweep_slabs_curved(G):
    _needs_gpu()
    spec = MeshSpec(degree=3, n_cells=(2, 3, 6), deform_amp=0.05, geometry="per_qpoint", seed=43)
    b = torch.from_numpy(uniform_vector(spec.n_dofs, 43)).cuda()
    x0 = torch.from_numpy(uniform_vector(spec.n_dofs, 44)).cuda()
    P, meshes, lb, sl = _setup(spec, G)
    ref = x0.clone()
    P.mesh_from_spec(spec).chebyshev_smooth(b, ref, 2.5, degree=3)
    xs = [x0[s].clone() for s in sl]
    bs = [b[s].clone() for s in sl]
    lb.run(lambda r: meshes[r].chebyshev_smooth(bs[r], xs[r], 2.5, degree=3))
    assert torch.equal(torch.cat(xs), ref)


@pytest.mark.parametrize("G", [2, 4])
def test_apply_and_dot_slabs(G):
    """dg_apply_laplace without DG_APPLY_HALO_READY (exchange inside) and dg_dot."""
    _needs_gpu()
    spec = MeshSpec(degree=4, n_cells=(3, 3, 8), bc=("periodic", "dirichlet", "periodic"), seed=45)
    u = torch.from_numpy(uniform_vector(spec.n_dofs, 45)).cuda()
    P, meshes, lb, sl = _setup(spec, G)
    single = P.mesh_from_spec(spec)
    ref = single.apply_laplace(u)
    us = [u[s].clone() for s in sl]
    ys = lb.run(lambda r: meshes[r].apply_laplace(us[r]))
    assert torch.equal(torch.cat(ys), ref)
    dots = lb.run(lambda r: meshes[r].dot(us[r], ys[r]))
    ref_dot = single.dot(u, ref)
    assert all(d == dots[0] for d in dots)
    assert abs(dots[0] - ref_dot) <= 1e-13 * abs(ref_dot)


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("inner", ["gl_jacobi", "fdm"])
def test_lanczos_slabs(G, inner):
    _needs_gpu()
    from oracle import fdm
    from oracle import smoother as sm
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    p = 3
    spec = MeshSpec(degree=p, n_cells=(3, 2, 6), bc=("dirichlet", "periodic", "dirichlet"), seed=46)
    P, meshes, lb, sl = _setup(spec, G)
    est = lb.run(lambda r: meshes[r].lanczos_lambda_max(inner, 15))
    assert all(e == est[0] for e in est)
    single = P.mesh_from_spec(spec).lanczos_lambda_max(inner, 15)
    assert abs(est[0] - single) <= 1e-12 * single
    om = mesh_from_spec(spec)
    H = SIPG(om, p)
    Pi = sm.GLJacobi(SIPG(om, p, "gl")) if inner == "gl_jacobi" else fdm.FDM(p, (1 / 3, 1 / 2, 1 / 6))
    ref = sm.lanczos_lambda_max(H.apply, Pi, spec.n_dofs, iters=15)
    assert abs(est[0] - ref) <= 1e-10 * ref


@pytest.mark.parametrize("G", [2, 3])
def test_pcg_slabs(G):
    _needs_gpu()
    from oracle.geometry import mesh_from_spec
    from oracle.sipg import SIPG
    p = 3
    spec = MeshSpec(degree=p, n_cells=(2, 2, 6), seed=47)
    b = torch.from_numpy(uniform_vector(spec.n_dofs, 47)).cuda()
    P, meshes, lb, sl = _setup(spec, G)
    bs = [b[s].clone() for s in sl]
    xs = [torch.zeros_like(bb) for bb in bs]
    res = lb.run(lambda r: meshes[r].pcg(bs[r], xs[r], 2.6, rel_tol=1e-10, max_iter=100, cheby_degree=3))
    assert all(rr == res[0] for rr in res)
    it, rel = res[0]
    assert rel <= 1e-10
    x1 = torch.zeros_like(b)
    it1, rel1 = P.mesh_from_spec(spec).pcg(b, x1, 2.6, rel_tol=1e-10, max_iter=100, cheby_degree=3)
    assert it == it1
    x = torch.cat(xs).cpu().numpy()
    assert np.linalg.norm(x - x1.cpu().numpy()) <= 1e-9 * np.linalg.norm(x1.cpu().numpy())
    A = SIPG(mesh_from_spec(spec), p).assemble()
    xs_ref = np.linalg.solve(A, b.cpu().numpy())
    assert np.linalg.norm(x - xs_ref) <= 1e-8 * np.linalg.norm(xs_ref)


def test_transport_errors():
    _needs_gpu()
    import paper_1907_08492_b200 as P
    spec = MeshSpec(degree=2, n_cells=(2, 2, 4))
    single = P.mesh_from_spec(spec)
    with pytest.raises(P.DgError, match="external"):
        single.set_transport(lambda *a: None, lambda x: x)
    m = P.mesh_from_spec(spec, rank=0, nranks=2)
    u = torch.zeros(m.n_local_dofs, dtype=torch.float64, device="cuda")
    with pytest.raises(P.DgError, match="UNSUPPORTED"):
        m.dot(u, u)

    def bad_halo(*a):
        raise RuntimeError("link down")
    m.set_transport(bad_halo, lambda x: x)
    with pytest.raises(P.DgError, match="transport failed"):
        m.apply_laplace(u)
