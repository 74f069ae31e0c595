"""Pins of the FDM oracle (oracle/fdm.py, Eqs. (13)-(15)).

The 1D interior-element matrices and Eq. (14) are checked against the independent 3D
naive quadrature of oracle/sipg.py: the diagonal block of an interior cell of the
assembled SIPG matrix must equal A^(K) (PAPER.md:2141-2145 states this form for
Cartesian cells), and the FDM inverse must invert it exactly.  Boundary cells use the
interior matrices, so there the preconditioner is not exact.
"""
import numpy as np
import pytest

from oracle import fdm
from oracle.geometry import mesh_from_spec
from oracle.sipg import SIPG
from synthetic.configs import MeshSpec


def _block(p, ncells, box_hi, cell):
    spec = MeshSpec(degree=p, n_cells=ncells, seed=0, box_hi=box_hi)
    m = mesh_from_spec(spec)
    n3 = (p + 1) ** 3
    c = int(m.cell_id(np.array([cell]))[0])
    U = np.zeros((m.ncells * n3, n3))
    U[c * n3 + np.arange(n3), np.arange(n3)] = 1.0          # unit vectors of cell c
    AKK = SIPG(m, p).apply(U, cells=[c])                     # rows of cell c: A_KK
    return AKK, tuple(bh / nc for bh, nc in zip(box_hi, ncells))


@pytest.mark.parametrize("p", [2, 3, 4, 5])
def test_interior_block_equals_kronecker_cell_matrix(p):
    AKK, h = _block(p, (3, 3, 3), (1.0, 1.0, 1.0), (1, 1, 1))
    AK = fdm.cell_matrix(p, h)
    assert np.abs(AKK - AK).max() <= 1e-13 * np.abs(AK).max()


@pytest.mark.parametrize("p", [2, 3, 5])
def test_fdm_inverts_interior_block_anisotropic(p):
    AKK, h = _block(p, (3, 3, 3), (1.0, 0.7, 1.9), (1, 1, 1))
    P = fdm.FDM(p, h)
    n3 = (p + 1) ** 3
    X = np.stack([P(AKK[:, j]) for j in range(n3)], 1)      # P^-1 A_KK
    assert np.abs(X - np.eye(n3)).max() <= 1e-12


def test_eigenpairs_and_gl_basis():
    for basis in ("hermite", "gl"):
        L, M = fdm.interior_1d(4, 0.25, basis)
        P = fdm.FDM(4, (0.25,) * 3, basis)
        Z, lam = P.Z[0], P.lam[0]
        assert np.abs(Z.T @ M @ Z - np.eye(5)).max() < 1e-12
        assert np.abs(L @ Z - M @ Z * lam).max() < 1e-10 * np.abs(L).max()
        assert lam.min() > 0                                  # interior block is SPD


def test_boundary_cell_is_approximate():
    """Corner cell under mirror BCs: the interior matrices are not its exact block."""
    AKK, h = _block(3, (3, 3, 3), (1.0, 1.0, 1.0), (0, 0, 0))
    P = fdm.FDM(3, h)
    X = np.stack([P(AKK[:, j]) for j in range(64)], 1)
    assert np.abs(X - np.eye(64)).max() > 1e-3
