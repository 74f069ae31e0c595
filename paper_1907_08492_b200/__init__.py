"""paper_1907_08492_b200 — B200-native (sm_100a, fp64) matrix-free SIPG in the
Hermite-like basis of arXiv 1907.08492.

The product is the C-ABI library libdg_b200.so (include/dg.h); this package
is its thin Python binding.  Importing it loads the library and fails loudly if
it has not been built (`python -m paper_1907_08492_b200.build`).
"""
from ._lib import LIB_PATH, lib  # noqa: F401
from .api import (APPLY_HALO_READY, APPLY_QUADRATURE, DgError, Mesh, get_nccl_unique_id,  # noqa: F401
                  halo_pack_host, measure_peak, mesh_from_spec, slab_plan, tables_1d,
                  version)
