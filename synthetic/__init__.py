"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no basis, quadrature, geometry
or operator code).  It only defines the BASELINE.json workload shapes
(SURVEY.md §8(d) "Synthetic inputs") and draws seeded random vectors, so that
the oracle (``oracle/``) and the product (``paper_1907_08492_b200``) are fed the
same bytes (SURVEY.md §8(c) reading 17).
"""
from .configs import CONFIGS, MeshSpec, config, c4_spec
from .vectors import uniform_vector

__all__ = ["CONFIGS", "MeshSpec", "config", "c4_spec", "uniform_vector"]
