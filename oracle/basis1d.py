"""Oracle: 1D quadrature rules and bases, in 50-digit mpmath, rounded to fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows PAPER.md §4.1 "Construction of the basis" step by
step, in the paper's notation, on the reference interval (0,1):
  step 1 (p=3, generalised for p>3 by step 3b): phi_0 = alpha_0 (xi - xi_1) B,
         phi_1 = w_1 xi B, with B = prod_l (xi - r_l) (xi - 1)^2;
         xi_1 from int_0^1 phi_0 phi_1 = 0 (linear in xi_1);
         alpha_0 from phi_0(0) = 1; w_1 from phi_1'(0) = -phi_0'(0)
         (Eq. (9)).
  step 2 (p<=2): p=1 Lagrange {1-xi, xi}; p=2 {(1-xi)^2, 2xi(1-xi), xi^2}
         (Appendix A).
  step 3a: interior nodes = roots of the Jacobi polynomial P^{4,4}_{p-3} on (0,1)
         (PAPER.md:637-644); bubbles xi^2 (1-xi)^2 prod_{m != l}(xi - r_m),
         normalised to 1 at their node r_l, ordered by increasing r_l
         (SURVEY.md §8(c) reading 2, confirmed by Appendix A p=4,5).
  mirror: phi_{p-i}(xi) = phi_i(1 - xi).
The nodal Gauss-Lobatto basis is the Lagrange basis on
{0, roots of P_p', 1} mapped to (0,1).

Polynomials are held as mpmath coefficient lists (low -> high) at 50 digits so
that the fp64 tables are correctly rounded even at p=8 (SURVEY.md finding 3:
fp64 monomial evaluation drifts to 1e-12 at p=8).
"""
from functools import lru_cache

import mpmath as mp
import numpy as np

DPS = 50


class Poly:
    """Polynomial with mpmath coefficients c[k] (coefficient of xi^k)."""

    def __init__(self, coeffs):
        self.c = [mp.mpf(x) for x in coeffs]

    @staticmethod
    def from_roots(scale, roots):
        c = [mp.mpf(scale)]
        for r in roots:
            r = mp.mpf(r)
            nc = [mp.mpf(0)] * (len(c) + 1)
            for k, a in enumerate(c):
                nc[k + 1] += a
                nc[k] -= a * r
            c = nc
        return Poly(c)

    def __call__(self, x):
        x = mp.mpf(x)
        acc = mp.mpf(0)
        for a in reversed(self.c):
            acc = acc * x + a
        return acc

    def deriv(self):
        return Poly([k * self.c[k] for k in range(1, len(self.c))] or [0])

    def __mul__(self, other):
        c = [mp.mpf(0)] * (len(self.c) + len(other.c) - 1)
        for i, a in enumerate(self.c):
            for j, b in enumerate(other.c):
                c[i + j] += a * b
        return Poly(c)

    def scale(self, s):
        return Poly([s * a for a in self.c])

    def integral01(self):
        return mp.fsum(a / (k + 1) for k, a in enumerate(self.c))

    def reflect(self):
        """q(xi) = self(1 - xi)."""
        out = Poly([0])
        # expand sum_k c_k (1 - xi)^k
        acc = [mp.mpf(0)] * len(self.c)
        for k, a in enumerate(self.c):
            # (1 - xi)^k = sum_m binom(k,m) (-xi)^m
            for m in range(k + 1):
                acc[m] += a * mp.binomial(k, m) * (-1) ** m
        out.c = acc
        return out


def _poly_roots(p: Poly):
    """Real roots of p, sorted (all roots of the orthogonal families are real)."""
    coeffs_hi_first = list(reversed(p.c))
    roots = mp.polyroots(coeffs_hi_first, maxsteps=400, extraprec=400)
    return sorted(mp.re(r) for r in roots)


def _jacobi_poly(m, alpha, beta):
    """P_m^{(alpha,beta)}(t) on [-1,1] by the standard three-term recurrence."""
    a, b = mp.mpf(alpha), mp.mpf(beta)
    P0 = Poly([1])
    if m == 0:
        return P0
    P1 = Poly([(a - b) / 2, (a + b + 2) / 2])
    for k in range(2, m + 1):
        c1 = 2 * k * (k + a + b) * (2 * k + a + b - 2)
        c2 = (2 * k + a + b - 1) * (a * a - b * b)
        c3 = (2 * k + a + b - 1) * (2 * k + a + b) * (2 * k + a + b - 2)
        c4 = 2 * (k + a - 1) * (k + b - 1) * (2 * k + a + b)
        t = Poly([0, 1])
        nxt_c = [mp.mpf(0)] * (k + 1)
        tp = t * P1
        for i, v in enumerate(tp.c):
            nxt_c[i] += c3 * v
        for i, v in enumerate(P1.c):
            nxt_c[i] += c2 * v
        for i, v in enumerate(P0.c):
            nxt_c[i] -= c4 * v
        P0, P1 = P1, Poly([v / c1 for v in nxt_c])
    return P1


def _to01(roots_pm1):
    return [(r + 1) / 2 for r in roots_pm1]


@lru_cache(maxsize=None)
def gauss_legendre(n: int):
    """n-point Gauss-Legendre rule on (0,1): (points, weights) as mpf tuples.

    Weights sum to 1 (reference interval (0,1))."""
    with mp.workdps(DPS):
        P = _jacobi_poly(n, 0, 0)
        t = _poly_roots(P)
        dP = P.deriv()
        w = [2 / ((1 - ti * ti) * dP(ti) ** 2) / 2 for ti in t]
        return tuple(_to01(t)), tuple(w)


@lru_cache(maxsize=None)
def gauss_lobatto_points(n: int):
    """n Gauss-Lobatto nodes on [0,1]: {0, roots of P_{n-1}', 1}."""
    with mp.workdps(DPS):
        if n == 2:
            return (mp.mpf(0), mp.mpf(1))
        dP = _jacobi_poly(n - 1, 0, 0).deriv()
        t = _poly_roots(dP)
        return tuple([mp.mpf(0)] + _to01(t) + [mp.mpf(1)])


@lru_cache(maxsize=None)
def jacobi44_roots(m: int):
    """The m roots of P^{4,4}_m mapped to (0,1), increasing."""
    with mp.workdps(DPS):
        if m == 0:
            return ()
        return tuple(_to01(_poly_roots(_jacobi_poly(m, 4, 4))))


@lru_cache(maxsize=None)
def hermite_like(p: int):
    """Hermite-like basis of degree p: (list of Poly, params dict)."""
    with mp.workdps(DPS):
        xi = Poly([0, 1])
        if p == 1:
            phis = [Poly([1, -1]), Poly([0, 1])]
            return phis, {"alpha1": mp.mpf(1)}
        if p == 2:
            phis = [Poly([1, -2, 1]), Poly([0, 2, -2]), Poly([0, 0, 1])]
            return phis, {"alpha1": mp.mpf(2)}
        r = jacobi44_roots(p - 3)
        B = Poly.from_roots(1, list(r) + [1, 1])            # prod (xi-r_l) (xi-1)^2
        # step 1/3b: xi_1 from int phi_0 phi_1 = 0, linear in xi_1:
        #   int (xi - xi_1) xi B^2 = 0  ->  xi_1 = int xi^2 B^2 / int xi B^2
        B2 = B * B
        xi1 = (xi * xi * B2).integral01() / (xi * B2).integral01()
        # alpha_0 from phi_0(0) = 1
        phi0_unit = Poly.from_roots(1, [xi1]) * B
        alpha0 = 1 / phi0_unit(0)
        phi0 = phi0_unit.scale(alpha0)
        # phi_1 = w1 xi B with phi_1'(0) = -phi_0'(0)
        phi1_unit = xi * B
        w1 = -phi0.deriv()(0) / phi1_unit.deriv()(0)
        phi1 = phi1_unit.scale(w1)
        # bubbles on the Jacobi roots, increasing node order
        bubbles = []
        for l, rl in enumerate(r):
            others = [rm for m_, rm in enumerate(r) if m_ != l]
            q = Poly.from_roots(1, [0, 0, 1, 1] + others)
            bubbles.append(q.scale(1 / q(rl)))
        phis = [phi0, phi1] + bubbles + [phi1.reflect(), phi0.reflect()]
        params = {"xi1": xi1, "alpha0": alpha0, "w1": w1,
                  "alpha1": phi1.deriv()(0), "roots": r}
        return phis, params


@lru_cache(maxsize=None)
def gl_lagrange(p: int):
    """Nodal Lagrange basis on the p+1 Gauss-Lobatto points of [0,1]."""
    with mp.workdps(DPS):
        x = gauss_lobatto_points(p + 1)
        phis = []
        for i, xi_ in enumerate(x):
            others = [xj for j, xj in enumerate(x) if j != i]
            q = Poly.from_roots(1, others)
            phis.append(q.scale(1 / q(xi_)))
        return phis


def basis_polys(p: int, basis: str):
    if basis == "hermite":
        return hermite_like(p)[0]
    if basis == "gl":
        return gl_lagrange(p)
    raise ValueError(basis)


def _f64(m):
    return np.array([[float(v) for v in row] for row in m], dtype=np.float64)


@lru_cache(maxsize=None)
def _tables(p: int, basis: str):
    with mp.workdps(DPS):
        n = p + 1
        phis = basis_polys(p, basis)
        dphis = [f.deriv() for f in phis]
        xq, wq = gauss_legendre(n)
        S = [[phis[j](xq[q]) for j in range(n)] for q in range(n)]
        DS = [[dphis[j](xq[q]) for j in range(n)] for q in range(n)]
        t = {
            "xq": np.array([float(v) for v in xq]),
            "wq": np.array([float(v) for v in wq]),
            "S": _f64(S),             # S[q][j]  = phi_j(xi_q)
            "DS": _f64(DS),           # DS[q][j] = phi_j'(xi_q)
            "v0": np.array([float(f(0)) for f in phis]),
            "v1": np.array([float(f(1)) for f in phis]),
            "d0": np.array([float(f(0)) for f in dphis]),
            "d1": np.array([float(f(1)) for f in dphis]),
        }
        return t


def tables(p: int, basis: str = "hermite"):
    """fp64 tables for the oracle's naive quadrature (copies)."""
    return {k: v.copy() for k, v in _tables(p, basis).items()}


def eval_basis(p: int, basis: str, x):
    """(values, derivatives) of all n basis functions at points x: shape (len(x), n)."""
    with mp.workdps(DPS):
        phis = basis_polys(p, basis)
        dphis = [f.deriv() for f in phis]
        V = [[f(xx) for f in phis] for xx in x]
        D = [[f(xx) for f in dphis] for xx in x]
        return _f64(V), _f64(D)


@lru_cache(maxsize=None)
def _T(p: int):
    with mp.workdps(DPS):
        n = p + 1
        xgl = gauss_lobatto_points(n)
        phis = hermite_like(p)[0]
        T = mp.matrix([[phis[j](xgl[i]) for j in range(n)] for i in range(n)])
        Ti = T ** -1
        return (_f64([[T[i, j] for j in range(n)] for i in range(n)]),
                _f64([[Ti[i, j] for j in range(n)] for i in range(n)]))


def change_matrix(p: int):
    """T[i][j] = phi_j^H(x_i^GL) (values of the Hermite-like basis at the GL
    nodes, SURVEY.md §8(c) reading 11) and T^{-1}, both rounded from 50 digits."""
    T, Ti = _T(p)
    return T.copy(), Ti.copy()


def mass_matrix_mp(p: int, basis: str):
    """Exact 1D mass matrix int_0^1 phi_i phi_j in mpmath (Table 1)."""
    with mp.workdps(DPS):
        phis = basis_polys(p, basis)
        n = p + 1
        return mp.matrix([[(phis[i] * phis[j]).integral01() for j in range(n)]
                          for i in range(n)])


def mass_condition(p: int, basis: str) -> float:
    """lambda_max / lambda_min of the 1D mass matrix (tab:condition_mass)."""
    with mp.workdps(DPS):
        M = mass_matrix_mp(p, basis)
        ev = mp.eigsy(M, eigvals_only=True)
        ev = sorted(ev)
        return float(ev[-1] / ev[0])
