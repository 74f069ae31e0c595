"""Host-only checks of the C ABI (no GPU): the library loads, exports every entry
point include/dg.h declares, and its host-built 1D tables equal the oracle's
(independently constructed in 50-digit mpmath) to rounding."""
import os
import re

import numpy as np
import pytest

from oracle import basis1d

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "dg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_1907_08492_b200 as P
    L = P.lib()
    names = _declared()
    assert "dg_apply_laplace" in names and "dg_mesh_setup" in names
    for name in names:
        assert hasattr(L, name), name
    nm = os.popen(f"nm -D --defined-only {P.LIB_PATH}").read()
    for name in names:
        assert re.search(rf"\bT {name}\b", nm), name


def test_version_and_error_paths():
    import paper_1907_08492_b200 as P
    assert "sm_100a" in P.version()
    with pytest.raises(P.DgError, match="DG_ERR_PARAM"):
        P.Mesh(degree=0, n_cells=(2, 2, 2))
    with pytest.raises(P.DgError, match="DG_ERR_PARAM"):
        P.Mesh(degree=3, n_cells=(2, 2, 2), box_lo=(0, 1, 0), box_hi=(1, 1, 1))
    with pytest.raises(P.DgError, match="DG_ERR_PARAM"):
        P.tables_1d(9)


@pytest.mark.parametrize("p", range(1, 9))
@pytest.mark.parametrize("basis", ["hermite", "gl"])
def test_host_tables_match_oracle(p, basis):
    import paper_1907_08492_b200 as P
    t = P.tables_1d(p, basis)
    o = basis1d.tables(p, basis)
    for k in ("xq", "wq", "S", "DS", "v0", "v1", "d0", "d1"):
        np.testing.assert_allclose(np.asarray(t[k]).reshape(o[k].shape), o[k], rtol=2e-16, atol=1e-28)
    if basis == "hermite":
        T, Ti = basis1d.change_matrix(p)
        np.testing.assert_allclose(np.asarray(t["T"]).reshape(T.shape), T, rtol=2e-16, atol=1e-28)
        np.testing.assert_allclose(np.asarray(t["Tinv"]).reshape(Ti.shape), Ti, rtol=1e-15, atol=1e-15)


def test_binding_checks_host_array_lengths():
    """The library reads 9 (user_inv_jac) / 6 (user_penalty) doubles per owned cell from raw
    host pointers and cannot check the length; the binding does, before dg_mesh_setup."""
    import paper_1907_08492_b200 as P
    with pytest.raises(ValueError, match="user_inv_jac"):
        P.Mesh(degree=2, n_cells=(2, 2, 2), geometry="per_cell", user_inv_jac=np.ones(9 * 8 - 1))
    with pytest.raises(ValueError, match="user_penalty"):
        P.Mesh(degree=2, n_cells=(2, 2, 3), user_penalty=np.ones(6 * 12 + 6))
    with pytest.raises(ValueError, match="user_penalty"):   # rank 1 of 2 owns planes [1, 3)
        P.Mesh(degree=2, n_cells=(2, 2, 3), user_penalty=np.ones(6 * 4), rank=1, nranks=2)
