"""ctypes loader for libdg_b200.so (the CUDA library built in-tree by build.py).

There is no fallback: if the shared library is missing or cannot be loaded the
import fails loudly (the product path never routes through the CPU oracle).
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdg_b200.so")


class DgDesc(ctypes.Structure):
    _fields_ = [
        ("degree", ctypes.c_int32),
        ("basis", ctypes.c_int32),
        ("n_cells", ctypes.c_int32 * 3),
        ("box_lo", ctypes.c_double * 3),
        ("box_hi", ctypes.c_double * 3),
        ("linear_map", ctypes.c_double * 9),
        ("deform_amp", ctypes.c_double),
        ("geometry", ctypes.c_int32),
        ("bc", ctypes.c_int32 * 3),
        ("penalty_factor", ctypes.c_double),
        ("user_inv_jac", ctypes.POINTER(ctypes.c_double)),
        ("user_penalty", ctypes.POINTER(ctypes.c_double)),
        ("rank", ctypes.c_int32),
        ("nranks", ctypes.c_int32),
        ("nccl_unique_id", ctypes.c_void_p),
        ("stream", ctypes.c_void_p),
    ]


HALO_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double))


class DgTransport(ctypes.Structure):
    _fields_ = [("halo", HALO_FN), ("allreduce_sum", ALLREDUCE_FN), ("user", ctypes.c_void_p)]


SYMBOLS = {
    "dg_set_transport": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(DgTransport)]),
    # name: (restype, argtypes)
    "dg_last_error": (ctypes.c_char_p, []),
    "dg_version": (ctypes.c_char_p, []),
    "dg_get_nccl_unique_id": (ctypes.c_int, [ctypes.c_void_p]),
    "dg_mesh_setup": (ctypes.c_int, [ctypes.POINTER(DgDesc), ctypes.POINTER(ctypes.c_void_p)]),
    "dg_mesh_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "dg_mesh_query": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64),
                                     ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int32),
                                     ctypes.POINTER(ctypes.c_int32)]),
    "dg_halo_exchange": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "dg_apply_laplace": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_int32, ctypes.c_void_p]),
    "dg_basis_change": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p]),
    "dg_chebyshev_smooth": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_int32, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_double, ctypes.c_int32,
                                           ctypes.c_void_p]),
    "dg_inverse_diagonal": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
                                           ctypes.c_void_p]),
    "dg_kernel_launch_count": (ctypes.c_int64, [ctypes.c_void_p]),
    "dg_measure_peak": (ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p]),
    "dg_slab_plan": (ctypes.c_int, [ctypes.c_int32] * 6 + [ctypes.POINTER(ctypes.c_int32)]),
    "dg_halo_pack_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]),
    "dg_mesh_query_halo": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64),
                                          ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]),
    "dg_halo_pack": (ctypes.c_int, [ctypes.c_void_p] * 5),
    "dg_halo_set": (ctypes.c_int, [ctypes.c_void_p] * 4),
    "dg_tables_1d": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                    ctypes.c_void_p, ctypes.c_int64]),
    "dg_apply_preconditioner": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_void_p]),
    "dg_dot": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.POINTER(ctypes.c_double), ctypes.c_void_p]),
    "dg_lanczos_lambda_max": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                             ctypes.POINTER(ctypes.c_double), ctypes.c_void_p]),
    "dg_apply_laplace_f32": (ctypes.c_int, [ctypes.c_void_p] * 4),
    "dg_apply_laplace_host": (ctypes.c_int, [ctypes.c_void_p] * 4),
    "dg_chebyshev_smooth_f32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_int32, ctypes.c_double,
                                               ctypes.c_double, ctypes.c_double, ctypes.c_int32,
                                               ctypes.c_void_p]),
    "dg_basis_change_f32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p]),
    "dg_pcg_mixed": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                    ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                    ctypes.POINTER(ctypes.c_double), ctypes.c_void_p]),
    "dg_pcg": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                              ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                              ctypes.c_double, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                              ctypes.POINTER(ctypes.c_double), ctypes.c_void_p]),
}

_lib = None


def lib():
    """Load libdg_b200.so (once) and declare every exported entry point."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          "`python -m paper_1907_08492_b200.build` (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    for name, (res, args) in SYMBOLS.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L
