"""The opt-in kernel variants (selected by environment variables the library reads once per
process) against the oracle, each in its own subprocess (tests/_variant_check.py): the
k_quad general kernel, the n = 5/6/8 alternates of k_kron4, the other output path of
k_kron4, the z-first basis change at every degree, the L2-prefetch settings, the i-plane
kernel k_kron6 on and off, and the n = 3 cell-per-thread kernel k_kron3c off (DG_K3C=0, so
that the n = 3 variants of k_kron4 / k_kron6 are the ones checked).  The defaults are covered
by test_gpu_parity.py."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

VARIANTS = [
    ({"DG_QUAD": "1"}, "3", True),
    ({"DG_K4_ALT": "44"}, "4,5,7", False),   # alternates at n = 5, 6, 8 (bits n-3)
    ({"DG_K4_ALT": "1", "DG_K3C": "0"}, "2", False),   # n = 3 alternate of k_kron4 (padded threads)
    ({"DG_K4_ALT5": "0"}, "4", False),       # n = 5: round 1's unpadded configuration
    ({"DG_K4_ALT7": "0"}, "6", False),       # n = 7: round 1's unpadded configuration
    ({"DG_K4_OUT": "0"}, "3,5", False),
    ({"DG_K4_OUT": "1", "DG_K3C": "0"}, "2,4", False),
    ({"DG_BCHG": "4"}, "1,3,4,5,6,7", False),
    ({"DG_BCHG": "1"}, "2,8", False),
    ({"DG_L2PF": "0"}, "5", False),
    ({"DG_L2PF": "2"}, "4", False),
    ({"DG_L2PF": "3"}, "3,6", False),
    ({"DG_K6": "255", "DG_K3C": "0"}, "2,3,4,5", False),   # k_kron6 i-plane matvec + Chebyshev for n = 3..6
    ({"DG_K6": "0", "DG_K3C": "0"}, "2,3,4,5", False),     # k_kron4 for every n
    ({"DG_L2PF": "0", "DG_K3C": "1"}, "2", False),          # k_kron3c (the n = 3 default) without L2 prefetch
    ({"DG_CHEBY_GLT": "0"}, "3,4", False),     # the direct GL-Jacobi step (no transformed residual)
    ({"DG_CHEBY_GLT": "9", "DG_K3C": "0"}, "2,5", False),   # transformed-residual step at n = 3 and 6 (bits n-3)
]


@pytest.mark.parametrize("env,degrees,curved", VARIANTS,
                         ids=[",".join(f"{k}={v}" for k, v in e.items()) for e, _, _ in VARIANTS])
def test_variant_parity(env, degrees, curved):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [sys.executable, os.path.join(HERE, "_variant_check.py"), degrees] + (["curved"] if curved else [])
    r = subprocess.run(cmd, env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


# Basis change (a12): the three kernels (DG_BCHG = 1 block-staged k_bchg, 4 z-first k_bchg4 via
# _variant_check above, 5 warp-private pipelined k_bchgw in its four line modes and two plane modes) and the per-n
# default mix, each at p = 1..8, all four ops, in place and out of place, fp64 and fp32
# (tests/_bchg_check.py).  DG_BCHGW_GRID=2 makes every warp stream many tiles through its slots.
BCHG_VARIANTS = [
    {"DG_BCHG": "5", "DG_BCHGW_MODE": "0", "DG_BCHGW_GRID": "2"},
    {"DG_BCHG": "5", "DG_BCHGW_MODE": "1", "DG_BCHGW_GRID": "2"},
    {"DG_BCHG": "5", "DG_BCHGW_MODE": "2", "DG_BCHGW_GRID": "2"},
    {"DG_BCHG": "5", "DG_BCHGW_MODE": "3", "DG_BCHGW_GRID": "2"},
    {"DG_BCHG": "5", "DG_BCHGW_MODE": "4", "DG_BCHGW_GRID": "2"},   # plane mode (k_bchgp), 3 slots
    {"DG_BCHG": "5", "DG_BCHGW_MODE": "6", "DG_BCHGW_GRID": "2"},   # plane mode, 2 slots
    {"DG_BCHG": "5"},
    {"DG_BCHG": "1"},
    {"DG_BCHGW_GRID": "2"},
    {},
]


@pytest.mark.parametrize("env", BCHG_VARIANTS,
                         ids=[",".join(f"{k}={v}" for k, v in e.items()) or "default" for e in BCHG_VARIANTS])
def test_basis_change_kernels(env):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [sys.executable, os.path.join(HERE, "_bchg_check.py")]
    r = subprocess.run(cmd, env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def test_plane_probe_runs():
    """The design probe of DESIGN.md §11 (dg_measure_peak kind 10 + n, csrc/k_probe_plane.cu) launches
    and returns a finite positive rate; bad kinds are rejected."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1907_08492_b200 as P
    for kind in ("plane_probe_n4", "plane_probe_nb_n4"):
        v = P.measure_peak(kind)
        assert v > 1.0 and v < 1e4
    import ctypes
    from paper_1907_08492_b200._lib import lib
    x = ctypes.c_double()
    assert lib().dg_measure_peak(9, ctypes.byref(x), None) != 0
    assert lib().dg_measure_peak(19, ctypes.byref(x), None) != 0
