"""Seeded fp64 input vectors, i.i.d. uniform on [-1, 1).

The paper does not specify input data (it benchmarks random-free throughput,
PAPER.md:1112-1120); BASELINE.json fixes "fp64 vector uniform[-1,1] seed s".
numpy's PCG64 stream is used so both sides can regenerate identical bytes.
"""
import numpy as np


def uniform_vector(n: int, seed: int) -> np.ndarray:
    """n doubles drawn i.i.d. from U[-1, 1) with numpy.random.default_rng(seed)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, size=int(n))
