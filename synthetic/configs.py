"""BASELINE.json workload shapes C1..C5 (SURVEY.md §8 preamble and §8(d)).

Plain data only: degree, cell counts, box, map parameters, boundary kinds and
seeds.  Everything numeric about the method lives in ``oracle/`` (test side)
or in the CUDA library (product side).
"""
from dataclasses import dataclass, field, replace
from typing import Tuple


@dataclass(frozen=True)
class MeshSpec:
    degree: int
    n_cells: Tuple[int, int, int]
    basis: str = "hermite"             # "hermite" | "gl"
    box_lo: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    box_hi: Tuple[float, float, float] = (1.0, 1.0, 1.0)
    linear_map: Tuple[float, ...] = (1.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0)
    deform_amp: float = 0.0            # x_i += amp*sin(2 pi X_j) sin(2 pi X_k), cyclic
    geometry: str = "constant"         # "constant" | "per_cell" | "per_qpoint"
    bc: Tuple[str, str, str] = ("dirichlet", "dirichlet", "dirichlet")  # or "periodic"
    penalty_factor: float = 1.0
    seed: int = 0

    @property
    def n(self) -> int:
        return self.degree + 1

    @property
    def n_cells_total(self) -> int:
        return self.n_cells[0] * self.n_cells[1] * self.n_cells[2]

    @property
    def n_dofs(self) -> int:
        return self.n_cells_total * self.n ** 3

    def with_(self, **kw) -> "MeshSpec":
        return replace(self, **kw)


# C4: N = round(480/(p+1)) cells per direction, 108-113 M DoF.
C4_N = {2: 160, 3: 120, 4: 96, 5: 80, 6: 69, 7: 60, 8: 53}


def c4_spec(p: int) -> MeshSpec:
    N = C4_N[p]
    return MeshSpec(degree=p, n_cells=(N, N, N), seed=10 + p)


CONFIGS = {
    # C1: p=3 on 4^3 Cartesian cells of [0,1]^3, 4096 DoF, seed 0
    "C1": MeshSpec(degree=3, n_cells=(4, 4, 4), seed=0),
    # C2: p=4 on 32^3 Cartesian cells, 4.1M DoF, seed 1 (Hermite vs nodal GL)
    "C2": MeshSpec(degree=4, n_cells=(32, 32, 32), seed=1),
    "C2_GL": MeshSpec(degree=4, n_cells=(32, 32, 32), basis="gl", seed=1),
    # C3: p=5 on 48^3 curved cells, amp 0.05, per-q-point geometry, seed 2
    "C3": MeshSpec(degree=5, n_cells=(48, 48, 48), deform_amp=0.05,
                   geometry="per_qpoint", seed=2),
    # C5: p=5 on 128^3 Cartesian cells, 453M DoF, seed 4
    "C5": MeshSpec(degree=5, n_cells=(128, 128, 128), seed=4),
}
for _p in C4_N:
    CONFIGS[f"C4_p{_p}"] = c4_spec(_p)


def config(name: str) -> MeshSpec:
    return CONFIGS[name]
