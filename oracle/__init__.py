"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct fp64 CPU implementation of what the hot path
of arXiv 1907.08492 computes.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.  The
product library (``paper_1907_08492_b200``) never imports, links or calls it,
and it shares no code with the CUDA path (SURVEY.md §1 "CPU oracle").

Modules
  basis1d    1D Gauss rules and the Hermite-like / Gauss-Lobatto bases, built in
             50-digit mpmath from the construction steps.
  geometry   the analytic mesh map and its Jacobian.
  sipg       naive element-wise SIPG quadrature, Eq. (1)/(3) (no sum
             factorisation, all n^3 basis functions summed explicitly).
  smoother   basis change T^{x3}, GL inverse diagonal, Chebyshev recurrence
             (Eqs. (11), (12)).

Parity status: every function is pinned by tests under tests/test_oracle_*.py
against paper-printed values, closed forms or independent constructions.  The
non-Cartesian geometry (the J^{-T} metric of Eq. (3), normals and areas of Eq. (1))
is pinned by tests/test_oracle_brute.py: a 40-digit mpmath face-wise bilinear form
with a numerically differentiated map, SIPG consistency of a mapped bubble on affine
bricks, and the single-cell energy identity that fixes the curved-face penalty to the
documented mean of A_F/V_K of both sides (SURVEY.md §8(c) reading 5; R5 —
the paper does not choose mean vs max, the pin holds the oracle to the documented
choice).  tools/oracle_mutants.py shows those pins fail for eight plausible mistakes.
"""
