"""Thin Python binding of the dg_b200 C ABI (include/dg.h).

Argument marshalling only: torch tensors provide device memory and the current
CUDA stream; every step of the hot path runs in the library's sm_100a kernels.
Names follow the C ABI (dg_mesh_setup -> Mesh, dg_apply_laplace -> apply_laplace, ...).
"""
import ctypes

import torch

from ._lib import ALLREDUCE_FN, HALO_FN, DgDesc, DgTransport, lib

DG_OK = 0
STATUS = {0: "DG_OK", 1: "DG_ERR_PARAM", 2: "DG_ERR_NUMERIC", 3: "DG_ERR_CUDA",
          4: "DG_ERR_NCCL", 5: "DG_ERR_UNSUPPORTED"}
BASIS = {"hermite": 0, "gl": 1}
GEOM = {"constant": 0, "per_cell": 1, "per_qpoint": 2}
BC = {"dirichlet": 0, "periodic": 1}
BCHG = {"T": 0, "Tinv": 1, "TT": 2, "TinvT": 3}
INNER = {"gl_jacobi": 0, "point_jacobi": 1, "fdm": 2}
APPLY_HALO_READY = 1
APPLY_QUADRATURE = 2


class DgError(RuntimeError):
    def __init__(self, status, where):
        msg = lib().dg_last_error().decode()
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")
        self.status = status


def _check(st, where):
    if st != DG_OK:
        raise DgError(st, where)


def _stream(stream):
    if stream is None:
        if not torch.cuda.is_available():
            return ctypes.c_void_p(0)
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, torch.cuda.Stream):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


def _ptr(t, n=None, name="tensor", dtype=None):
    dtype = torch.float64 if dtype is None else dtype
    if not isinstance(t, torch.Tensor) or t.dtype != dtype or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA {dtype} tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if n is not None and t.numel() < n:
        raise ValueError(f"{name} has {t.numel()} elements, need {n}")
    if t.data_ptr() % 16:
        raise ValueError(f"{name} must be 16-byte aligned (dg.h conventions); got a view at an odd offset")
    return ctypes.c_void_p(t.data_ptr())


def get_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().dg_get_nccl_unique_id(buf), "dg_get_nccl_unique_id")
    return buf.raw


def measure_peak(kind: str, stream=None) -> float:
    """'fp64' -> TFLOP/s of DFMA; 'copy' / 'read' -> GB/s; 'dmma' -> fp64 tensor-core TFLOP/s;
    'dmma+dfma' -> both interleaved; 'plane_probe_n<N>' (N = 3..8) -> GDoF/s of the pipelined-plane
    matvec proxy (see dg_measure_peak)."""
    v = ctypes.c_double()
    kinds = {"fp64": 0, "copy": 1, "read": 2, "dmma": 3, "dmma+dfma": 4}
    kinds.update({f"plane_probe_n{n}": 10 + n for n in range(3, 9)})
    kinds.update({f"plane_probe_nb_n{n}": 20 + n for n in range(3, 7)})   # with neighbour traffic
    _check(lib().dg_measure_peak(kinds[kind], ctypes.byref(v),
                                 _stream(stream)), "dg_measure_peak")
    return v.value


def version() -> str:
    return lib().dg_version().decode()


def tables_1d(degree: int, basis: str = "hermite", penalty_factor: float = 1.0):
    """Host-only: the 1D tables of the kernels (dict of numpy arrays), see dg.h."""
    import numpy as np
    n = degree + 1
    need = 6 * n + 9 * n * n
    out = (ctypes.c_double * need)()
    _check(lib().dg_tables_1d(degree, BASIS[basis], penalty_factor, out, need), "dg_tables_1d")
    a = np.frombuffer(out, dtype=np.float64).copy()
    names = [("xq", n), ("wq", n), ("S", n * n), ("DS", n * n), ("v0", n), ("v1", n), ("d0", n),
             ("d1", n), ("Mhat", n * n), ("Ahat", n * n), ("Lhat", n * n), ("Nm", n * n),
             ("Np", n * n), ("T", n * n), ("Tinv", n * n)]
    res, o = {}, 0
    for k, c in names:
        v = a[o:o + c]
        res[k] = v.reshape(n, n) if c == n * n and n > 1 else v
        o += c
    return res


def slab_plan(Nz, nranks, rank, bc_z="dirichlet", degree=3, basis="hermite"):
    """Host-only dg_slab_plan: dict(z_begin, z_end, lo_peer, hi_peer, NL)."""
    out = (ctypes.c_int32 * 6)()
    _check(lib().dg_slab_plan(int(Nz), int(nranks), int(rank), BC[bc_z], int(degree), BASIS[basis], out),
           "dg_slab_plan")
    return dict(z_begin=out[0], z_end=out[1], lo_peer=out[2], hi_peer=out[3], NL=out[4])


def halo_pack_host(u_slab, degree, basis, Nx, Ny, nz):
    """Host-only reference packer: (send_lo, send_hi) numpy arrays of a host slab."""
    import numpy as np
    u = np.ascontiguousarray(u_slab, dtype=np.float64)
    n = degree + 1
    NL = 2 if (basis == "hermite" and degree >= 2) else n
    cnt = Nx * Ny * NL * n * n
    lo = np.empty(cnt)
    hi = np.empty(cnt)
    _check(lib().dg_halo_pack_host(u.ctypes.data, degree, BASIS[basis], Nx, Ny, nz, lo.ctypes.data,
                                   hi.ctypes.data), "dg_halo_pack_host")
    return lo, hi


class Mesh:
    """dg_mesh_setup(...) handle.  All vectors are CUDA float64 tensors of n_local_dofs."""

    def __init__(self, degree, n_cells, basis="hermite", box_lo=(0.0, 0.0, 0.0),
                 box_hi=(1.0, 1.0, 1.0), linear_map=None, deform_amp=0.0, geometry="constant",
                 bc=("dirichlet", "dirichlet", "dirichlet"), penalty_factor=1.0,
                 user_inv_jac=None, user_penalty=None, rank=0, nranks=1, nccl_unique_id=None,
                 stream=None):
        L = lib()
        d = DgDesc()
        d.degree = int(degree)
        d.basis = BASIS[basis]
        for k in range(3):
            d.n_cells[k] = int(n_cells[k])
            d.box_lo[k] = float(box_lo[k])
            d.box_hi[k] = float(box_hi[k])
            d.bc[k] = BC[bc[k]]
        lm = linear_map if linear_map is not None else (1, 0, 0, 0, 1, 0, 0, 0, 1)
        for k in range(9):
            d.linear_map[k] = float(lm[k])
        d.deform_amp = float(deform_amp)
        d.geometry = GEOM[geometry]
        d.penalty_factor = float(penalty_factor)
        self._jac_keepalive = None
        if user_inv_jac is not None:
            import numpy as np
            arr = np.ascontiguousarray(user_inv_jac, dtype=np.float64).reshape(-1)
            nloc = int(n_cells[0]) * int(n_cells[1]) * self._local_planes(n_cells[2], rank, nranks)
            if arr.size != 9 * nloc:
                raise ValueError(f"user_inv_jac has {arr.size} doubles, need 9 per owned cell = {9 * nloc}")
            self._jac_keepalive = arr
            d.user_inv_jac = arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        self._pen_keepalive = None
        if user_penalty is not None:
            import numpy as np
            arr = np.ascontiguousarray(user_penalty, dtype=np.float64).reshape(-1)
            nloc = int(n_cells[0]) * int(n_cells[1]) * self._local_planes(n_cells[2], rank, nranks)
            if arr.size != 6 * nloc:
                raise ValueError(f"user_penalty has {arr.size} doubles, need 6 per owned cell = {6 * nloc}")
            self._pen_keepalive = arr
            d.user_penalty = arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        d.rank = int(rank)
        d.nranks = int(nranks)
        self._id_keepalive = None
        if nccl_unique_id is not None:
            self._id_keepalive = ctypes.create_string_buffer(bytes(nccl_unique_id), 128)
            d.nccl_unique_id = ctypes.cast(self._id_keepalive, ctypes.c_void_p)
        d.stream = _stream(stream).value
        h = ctypes.c_void_p()
        _check(L.dg_mesh_setup(ctypes.byref(d), ctypes.byref(h)), "dg_mesh_setup")
        self._h = h
        nl, ng = ctypes.c_int64(), ctypes.c_int64()
        zb, ze = ctypes.c_int32(), ctypes.c_int32()
        _check(L.dg_mesh_query(h, ctypes.byref(nl), ctypes.byref(ng), ctypes.byref(zb),
                               ctypes.byref(ze)), "dg_mesh_query")
        self.n_local_dofs, self.n_global_dofs = nl.value, ng.value
        self.z_begin, self.z_end = zb.value, ze.value
        self.degree = int(degree)
        self.n = self.degree + 1

    @staticmethod
    def _local_planes(Nz, rank, nranks):
        P = max(int(nranks), 1)
        r = int(rank)
        return (r + 1) * int(Nz) // P - r * int(Nz) // P

    # ------------------------------------------------------------------ lifetime
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().dg_mesh_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launch_count(self) -> int:
        return int(lib().dg_kernel_launch_count(self._h))

    def empty(self):
        return torch.empty(self.n_local_dofs, dtype=torch.float64, device="cuda")

    # ------------------------------------------------------------------ operators
    def halo_exchange(self, u, stream=None):
        _check(lib().dg_halo_exchange(self._h, _ptr(u, self.n_local_dofs, "u"), _stream(stream)),
               "dg_halo_exchange")

    def query_halo(self):
        c, lo, hi = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
        _check(lib().dg_mesh_query_halo(self._h, ctypes.byref(c), ctypes.byref(lo), ctypes.byref(hi)),
               "dg_mesh_query_halo")
        return dict(count=c.value, lo_peer=lo.value, hi_peer=hi.value)

    def halo_pack(self, u, send_lo=None, send_hi=None, stream=None):
        """External transport: the two send planes of u (device tensors)."""
        cnt = self.query_halo()["count"]
        if send_lo is None:
            send_lo = torch.empty(max(cnt, 1), dtype=torch.float64, device="cuda")
        if send_hi is None:
            send_hi = torch.empty(max(cnt, 1), dtype=torch.float64, device="cuda")
        _check(lib().dg_halo_pack(self._h, _ptr(u, self.n_local_dofs, "u"), _ptr(send_lo, cnt, "send_lo"),
                                  _ptr(send_hi, cnt, "send_hi"), _stream(stream)), "dg_halo_pack")
        return send_lo, send_hi

    def halo_set(self, recv_lo=None, recv_hi=None, stream=None):
        cnt = self.query_halo()["count"]
        lo = _ptr(recv_lo, cnt, "recv_lo") if recv_lo is not None else ctypes.c_void_p(0)
        hi = _ptr(recv_hi, cnt, "recv_hi") if recv_hi is not None else ctypes.c_void_p(0)
        _check(lib().dg_halo_set(self._h, lo, hi, _stream(stream)), "dg_halo_set")

    def set_transport(self, halo, allreduce_sum):
        """dg_set_transport (external mode): halo(send_lo, send_hi, recv_lo, recv_hi, count, stream)
        gets raw device pointers (int or None) and must fill the recv planes; allreduce_sum(x)
        returns the sum of the host float x over all ranks.  Exceptions become a non-zero
        status (DG_ERR_NCCL "transport failed").  halo=None removes the transport."""
        if halo is None:
            _check(lib().dg_set_transport(self._h, None), "dg_set_transport")
            self._transport = None
            return

        def _halo(user, slo, shi, rlo, rhi, count, stream):
            try:
                halo(slo, shi, rlo, rhi, int(count), stream)
                return 0
            except Exception:                      # noqa: BLE001 - reported as a status
                import traceback
                traceback.print_exc()
                return 1

        def _sum(user, val):
            try:
                val[0] = float(allreduce_sum(float(val[0])))
                return 0
            except Exception:                      # noqa: BLE001
                import traceback
                traceback.print_exc()
                return 1

        t = DgTransport(HALO_FN(_halo), ALLREDUCE_FN(_sum), None)
        self._transport = t                        # keeps the C callbacks alive
        _check(lib().dg_set_transport(self._h, ctypes.byref(t)), "dg_set_transport")

    def halo_set_raw(self, recv_lo_ptr, recv_hi_ptr, stream=None):
        """dg_halo_set with raw device pointers (for transports)."""
        _check(lib().dg_halo_set(self._h, ctypes.c_void_p(recv_lo_ptr or 0), ctypes.c_void_p(recv_hi_ptr or 0),
                                 _stream(stream)), "dg_halo_set")

    def apply_laplace(self, u, y=None, flags=0, stream=None):
        if y is None:
            y = self.empty()
        _check(lib().dg_apply_laplace(self._h, _ptr(u, self.n_local_dofs, "u"),
                                      _ptr(y, self.n_local_dofs, "y"), int(flags), _stream(stream)),
               "dg_apply_laplace")
        return y

    def apply_laplace_host(self, u, y=None, stream=None):
        """y = A u for HOST (CPU, ideally pinned) float64 tensors; the copies are overlapped with
        the kernels inside the library (dg_apply_laplace_host).  Returns when `stream` is
        synchronised by the caller (stream-ordered)."""
        if not isinstance(u, torch.Tensor) or u.dtype != torch.float64 or u.is_cuda or not u.is_contiguous():
            raise TypeError("u must be a contiguous CPU float64 tensor")
        if y is None:
            y = torch.empty(self.n_local_dofs, dtype=torch.float64, pin_memory=u.is_pinned())
        if y.dtype != torch.float64 or y.is_cuda or not y.is_contiguous() or y.numel() < self.n_local_dofs:
            raise TypeError("y must be a contiguous CPU float64 tensor of n_local_dofs")
        if u.numel() < self.n_local_dofs:
            raise ValueError("u too short")
        _check(lib().dg_apply_laplace_host(self._h, ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                                           _stream(stream)), "dg_apply_laplace_host")
        return y

    def apply_laplace_f32(self, u, y=None, stream=None):
        """y = A u in single precision (Cartesian meshes, single slab)."""
        f32 = torch.float32
        if y is None:
            y = torch.empty(self.n_local_dofs, dtype=f32, device="cuda")
        _check(lib().dg_apply_laplace_f32(self._h, _ptr(u, self.n_local_dofs, "u", f32),
                                          _ptr(y, self.n_local_dofs, "y", f32), _stream(stream)),
               "dg_apply_laplace_f32")
        return y

    def chebyshev_smooth_f32(self, b, x, lambda_max, degree=5, lo=0.06, hi=1.2, inner="gl_jacobi",
                             work2=None, stream=None):
        f32 = torch.float32
        if work2 is None:
            work2 = torch.empty(2 * self.n_local_dofs, dtype=f32, device="cuda")
        _check(lib().dg_chebyshev_smooth_f32(self._h, _ptr(b, self.n_local_dofs, "b", f32),
                                             _ptr(x, self.n_local_dofs, "x", f32),
                                             _ptr(work2, 2 * self.n_local_dofs, "work2", f32), int(degree),
                                             float(lambda_max), float(lo), float(hi), INNER[inner],
                                             _stream(stream)), "dg_chebyshev_smooth_f32")
        return x

    def basis_change(self, op, x, out=None, stream=None):
        if out is None:
            out = self.empty()
        _check(lib().dg_basis_change(self._h, BCHG[op], _ptr(x, self.n_local_dofs, "in"),
                                     _ptr(out, self.n_local_dofs, "out"), _stream(stream)),
               "dg_basis_change")
        return out

    def chebyshev_smooth(self, b, x, lambda_max, degree=5, lo=0.06, hi=1.2, inner="gl_jacobi",
                         work2=None, stream=None):
        if work2 is None:
            work2 = torch.empty(2 * self.n_local_dofs, dtype=torch.float64, device="cuda")
        _check(lib().dg_chebyshev_smooth(self._h, _ptr(b, self.n_local_dofs, "b"),
                                         _ptr(x, self.n_local_dofs, "x"),
                                         _ptr(work2, 2 * self.n_local_dofs, "work2"), int(degree),
                                         float(lambda_max), float(lo), float(hi), INNER[inner],
                                         _stream(stream)), "dg_chebyshev_smooth")
        return x

    def apply_preconditioner(self, r, z=None, inner="gl_jacobi", stream=None):
        """z = P^{-1} r for the inner preconditioner of the smoother (Eq. (12) / FDM)."""
        if z is None:
            z = self.empty()
        _check(lib().dg_apply_preconditioner(self._h, INNER[inner], _ptr(r, self.n_local_dofs, "r"),
                                             _ptr(z, self.n_local_dofs, "z"), _stream(stream)),
               "dg_apply_preconditioner")
        return z

    def dot(self, a, b, stream=None) -> float:
        """Global (all-rank) dot product on the GPU, deterministic two-level reduction."""
        out = ctypes.c_double()
        _check(lib().dg_dot(self._h, _ptr(a, self.n_local_dofs, "a"), _ptr(b, self.n_local_dofs, "b"),
                            ctypes.byref(out), _stream(stream)), "dg_dot")
        return out.value

    def lanczos_lambda_max(self, inner="gl_jacobi", iters=15, stream=None) -> float:
        """lambda_max(P^{-1}A) from `iters` Lanczos steps."""
        out = ctypes.c_double()
        _check(lib().dg_lanczos_lambda_max(self._h, INNER[inner], int(iters), ctypes.byref(out),
                                           _stream(stream)), "dg_lanczos_lambda_max")
        return out.value

    def pcg(self, b, x, lambda_max, rel_tol=1e-9, max_iter=500, cheby_degree=5, lo=0.06, hi=1.2,
            inner="gl_jacobi", stream=None):
        """CG with the Chebyshev sweep as preconditioner; x: in initial guess, out solution.
        Returns (iterations, relative residual)."""
        it = ctypes.c_int32()
        rr = ctypes.c_double()
        _check(lib().dg_pcg(self._h, _ptr(b, self.n_local_dofs, "b"), _ptr(x, self.n_local_dofs, "x"),
                            float(rel_tol), int(max_iter), int(cheby_degree), float(lambda_max), float(lo),
                            float(hi), INNER[inner], ctypes.byref(it), ctypes.byref(rr), _stream(stream)),
               "dg_pcg")
        return it.value, rr.value

    def basis_change_f32(self, op, x, out=None, stream=None):
        """fp32 basis change B^{x3} per cell (dg_basis_change_f32)."""
        f32 = torch.float32
        if out is None:
            out = torch.empty(self.n_local_dofs, dtype=f32, device="cuda")
        _check(lib().dg_basis_change_f32(self._h, BCHG[op], _ptr(x, self.n_local_dofs, "in", f32),
                                         _ptr(out, self.n_local_dofs, "out", f32), _stream(stream)),
               "dg_basis_change_f32")
        return out

    def pcg_mixed(self, b, x, lambda_max, rel_tol=1e-9, max_iter=500, cheby_degree=5, lo=0.06, hi=1.2,
                  inner="gl_jacobi", stream=None):
        """dg_pcg_mixed: fp64 CG around an fp32 Chebyshev preconditioner.  Returns (iterations,
        relative residual)."""
        it = ctypes.c_int32()
        rr = ctypes.c_double()
        _check(lib().dg_pcg_mixed(self._h, _ptr(b, self.n_local_dofs, "b"), _ptr(x, self.n_local_dofs, "x"),
                                  float(rel_tol), int(max_iter), int(cheby_degree), float(lambda_max), float(lo),
                                  float(hi), INNER[inner], ctypes.byref(it), ctypes.byref(rr), _stream(stream)),
               "dg_pcg_mixed")
        return it.value, rr.value

    def inverse_diagonal(self, inner="gl_jacobi", out=None, stream=None):
        if out is None:
            out = self.empty()
        _check(lib().dg_inverse_diagonal(self._h, INNER[inner], _ptr(out, self.n_local_dofs, "out"),
                                         _stream(stream)), "dg_inverse_diagonal")
        return out


def mesh_from_spec(spec, **kw) -> Mesh:
    """Mesh from a synthetic.MeshSpec (plain data)."""
    args = dict(degree=spec.degree, n_cells=spec.n_cells, basis=spec.basis, box_lo=spec.box_lo,
                box_hi=spec.box_hi, linear_map=spec.linear_map, deform_amp=spec.deform_amp,
                geometry=spec.geometry, bc=spec.bc, penalty_factor=spec.penalty_factor)
    args.update(kw)
    return Mesh(**args)
