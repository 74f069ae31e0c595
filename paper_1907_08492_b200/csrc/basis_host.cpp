// Host construction of the 1D bases and reference matrices in __float128.
//
// Hermite-like basis, Sec. 4.1 (lines 596-659), reference interval (0,1):
//   p=1: {1-x, x};  p=2: {(1-x)^2, 2x(1-x), x^2}   (Appendix A)
//   p>=3: B(x) = prod_l (x - r_l) (x-1)^2, r_l the roots of P^{4,4}_{p-3} on (0,1);
//         x1 = int x^2 B^2 / int x B^2          (int phi_0 phi_1 = 0)
//         phi_0 = a0 (x - x1) B,  phi_0(0) = 1
//         phi_1 = w1 x B,  phi_1'(0) = -phi_0'(0) (Eq. (9))
//         bubbles x^2 (1-x)^2 prod_{m!=l}(x - r_m) / (same at r_l), increasing r_l
//         phi_{p-i}(x) = phi_i(1-x)
// Nodal Gauss-Lobatto: Lagrange on {0, roots of P^{1,1}_{p-1}, 1}.
// 1D SIPG blocks for the Cartesian Kronecker form, Eq. (14).
#include "basis_host.h"

#include <algorithm>
#include <cmath>
#include <vector>

namespace dgb {
namespace {

typedef __float128 qr;

struct QPoly {
  std::vector<qr> c;  // c[k] * x^k
  QPoly() : c(1, 0) {}
  explicit QPoly(std::vector<qr> v) : c(std::move(v)) {}
  static QPoly monomial_root(qr r) { return QPoly({-r, 1}); }
  qr operator()(qr x) const {
    qr a = 0;
    for (int k = (int)c.size() - 1; k >= 0; --k) a = a * x + c[k];
    return a;
  }
  QPoly deriv() const {
    if (c.size() <= 1) return QPoly({0});
    std::vector<qr> d(c.size() - 1);
    for (size_t k = 1; k < c.size(); ++k) d[k - 1] = (qr)k * c[k];
    return QPoly(d);
  }
  QPoly operator*(const QPoly& o) const {
    std::vector<qr> r(c.size() + o.c.size() - 1, 0);
    for (size_t i = 0; i < c.size(); ++i)
      for (size_t j = 0; j < o.c.size(); ++j) r[i + j] += c[i] * o.c[j];
    return QPoly(r);
  }
  QPoly operator+(const QPoly& o) const {
    std::vector<qr> r(std::max(c.size(), o.c.size()), 0);
    for (size_t i = 0; i < c.size(); ++i) r[i] += c[i];
    for (size_t i = 0; i < o.c.size(); ++i) r[i] += o.c[i];
    return QPoly(r);
  }
  QPoly scaled(qr s) const {
    QPoly r = *this;
    for (auto& v : r.c) v *= s;
    return r;
  }
  qr integral01() const {
    qr s = 0;
    for (size_t k = 0; k < c.size(); ++k) s += c[k] / (qr)(k + 1);
    return s;
  }
  // q(x) = p(1-x)
  QPoly reflected() const {
    QPoly acc({0});
    QPoly one_minus_x({1, -1});
    QPoly pw({1});
    for (size_t k = 0; k < c.size(); ++k) {
      acc = acc + pw.scaled(c[k]);
      pw = pw * one_minus_x;
    }
    return acc;
  }
};

QPoly from_roots(qr scale, const std::vector<qr>& roots) {
  QPoly p({scale});
  for (qr r : roots) p = p * QPoly::monomial_root(r);
  return p;
}

qr qabs(qr x) { return x < 0 ? -x : x; }

// Jacobi P_m^{(a,b)} on [-1,1], monomial coefficients via the three-term recurrence.
QPoly jacobi(int m, qr a, qr b) {
  QPoly P0({1});
  if (m == 0) return P0;
  QPoly P1({(a - b) / 2, (a + b + 2) / 2});
  for (int k = 2; k <= m; ++k) {
    qr c1 = 2 * k * (k + a + b) * (2 * k + a + b - 2);
    qr c2 = (2 * k + a + b - 1) * (a * a - b * b);
    qr c3 = (2 * k + a + b - 1) * (2 * k + a + b) * (2 * k + a + b - 2);
    qr c4 = 2 * (k + a - 1) * (k + b - 1) * (2 * k + a + b);
    QPoly t = QPoly({0, 1}) * P1;
    std::vector<qr> nx(k + 1, 0);
    for (size_t i = 0; i < t.c.size(); ++i) nx[i] += c3 * t.c[i];
    for (size_t i = 0; i < P1.c.size(); ++i) nx[i] += c2 * P1.c[i];
    for (size_t i = 0; i < P0.c.size(); ++i) nx[i] -= c4 * P0.c[i];
    for (auto& v : nx) v /= c1;
    P0 = P1;
    P1 = QPoly(nx);
  }
  return P1;
}

// All (real, simple) roots in (-1,1) of a degree-m orthogonal polynomial: Newton
// with implicit deflation (Aberth-free, sequential), started from Chebyshev nodes.
std::vector<qr> real_roots(const QPoly& P, int m) {
  QPoly dP = P.deriv();
  std::vector<qr> roots;
  for (int k = 0; k < m; ++k) {
    qr x = (qr)std::cos(M_PI * (k + 0.75) / (m + 0.5));
    for (int it = 0; it < 200; ++it) {
      qr f = P(x), fp = dP(x);
      qr s = 0;
      for (qr r : roots) s += 1 / (x - r);
      qr dx = f / (fp - f * s);
      x -= dx;
      if (qabs(dx) < (qr)1e-32) break;
    }
    roots.push_back(x);
  }
  std::sort(roots.begin(), roots.end());
  return roots;
}

std::vector<qr> to01(const std::vector<qr>& r) {
  std::vector<qr> o;
  for (qr v : r) o.push_back((v + 1) / 2);
  return o;
}

void gauss(int n, std::vector<qr>& x, std::vector<qr>& w) {
  QPoly P = jacobi(n, 0, 0);
  std::vector<qr> t = real_roots(P, n);
  QPoly dP = P.deriv();
  x.clear();
  w.clear();
  for (qr ti : t) {
    qr d = dP(ti);
    x.push_back((ti + 1) / 2);
    w.push_back(1 / ((1 - ti * ti) * d * d));  // 2/((1-t^2)P'^2) / 2
  }
}

std::vector<QPoly> hermite_like(int p) {
  std::vector<QPoly> phi;
  if (p == 1) return {QPoly({1, -1}), QPoly({0, 1})};
  if (p == 2) return {QPoly({1, -2, 1}), QPoly({0, 2, -2}), QPoly({0, 0, 1})};
  std::vector<qr> r = p > 3 ? to01(real_roots(jacobi(p - 3, 4, 4), p - 3)) : std::vector<qr>();
  std::vector<qr> broots = r;
  broots.push_back(1);
  broots.push_back(1);
  QPoly B = from_roots(1, broots);
  QPoly B2 = B * B;
  QPoly x({0, 1});
  qr x1 = (x * x * B2).integral01() / (x * B2).integral01();
  QPoly phi0u = QPoly::monomial_root(x1) * B;
  QPoly phi0 = phi0u.scaled(1 / phi0u(0));
  QPoly phi1u = x * B;
  QPoly phi1 = phi1u.scaled(-phi0.deriv()(0) / phi1u.deriv()(0));
  phi.push_back(phi0);
  phi.push_back(phi1);
  for (size_t l = 0; l < r.size(); ++l) {
    std::vector<qr> rr = {0, 0, 1, 1};
    for (size_t m = 0; m < r.size(); ++m)
      if (m != l) rr.push_back(r[m]);
    QPoly q = from_roots(1, rr);
    phi.push_back(q.scaled(1 / q(r[l])));
  }
  phi.push_back(phi1.reflected());
  phi.push_back(phi0.reflected());
  return phi;
}

std::vector<qr> gl_points(int n) {
  std::vector<qr> x = {0};
  if (n > 2) {
    std::vector<qr> t = to01(real_roots(jacobi(n - 2, 1, 1), n - 2));
    x.insert(x.end(), t.begin(), t.end());
  }
  x.push_back(1);
  return x;
}

std::vector<QPoly> gl_lagrange(int p) {
  std::vector<qr> x = gl_points(p + 1);
  std::vector<QPoly> phi;
  for (int i = 0; i <= p; ++i) {
    std::vector<qr> others;
    for (int j = 0; j <= p; ++j)
      if (j != i) others.push_back(x[j]);
    QPoly q = from_roots(1, others);
    phi.push_back(q.scaled(1 / q(x[i])));
  }
  return phi;
}

// Gauss-Jordan inverse in quad precision.
std::vector<qr> inverse(std::vector<qr> A, int n) {
  std::vector<qr> I(n * n, 0);
  for (int i = 0; i < n; ++i) I[i * n + i] = 1;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (qabs(A[r * n + c]) > qabs(A[piv * n + c])) piv = r;
    for (int k = 0; k < n; ++k) {
      std::swap(A[c * n + k], A[piv * n + k]);
      std::swap(I[c * n + k], I[piv * n + k]);
    }
    qr d = A[c * n + c];
    for (int k = 0; k < n; ++k) {
      A[c * n + k] /= d;
      I[c * n + k] /= d;
    }
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      qr f = A[r * n + c];
      for (int k = 0; k < n; ++k) {
        A[r * n + k] -= f * A[c * n + k];
        I[r * n + k] -= f * I[c * n + k];
      }
    }
  }
  return I;
}

struct QTables {
  std::vector<qr> S, DS, v0, v1, d0, d1, M, A, L, Nm, Np;
};

// 1D SIPG pieces on the reference interval (h = 1), sigma_hat = (p+1)^2 * pf.
// Element-wise face terms (Eq. (1)) on a face with outward normal nu and
// physical derivative (nu/h) d/dxi, h = 1:
//   own-own   : sigma v_i v_j - 1/2 nu v_i d_j - 1/2 nu d_i v_j
//   own-neigh : -sigma v_i w_j - 1/2 nu v_i e_j + 1/2 nu d_i w_j   (w, e: neighbour trace)
QTables build_q(const std::vector<QPoly>& phi, const std::vector<qr>& xq,
                const std::vector<qr>& wq, qr sigma) {
  int n = (int)phi.size();
  QTables t;
  std::vector<QPoly> dphi;
  for (auto& f : phi) dphi.push_back(f.deriv());
  t.S.resize(n * n);
  t.DS.resize(n * n);
  for (int q = 0; q < n; ++q)
    for (int j = 0; j < n; ++j) {
      t.S[q * n + j] = phi[j](xq[q]);
      t.DS[q * n + j] = dphi[j](xq[q]);
    }
  for (int j = 0; j < n; ++j) {
    t.v0.push_back(phi[j](0));
    t.v1.push_back(phi[j](1));
    t.d0.push_back(dphi[j](0));
    t.d1.push_back(dphi[j](1));
  }
  t.M.assign(n * n, 0);
  t.A.assign(n * n, 0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      qr m = 0, a = 0;
      for (int q = 0; q < n; ++q) {
        m += wq[q] * t.S[q * n + i] * t.S[q * n + j];
        a += wq[q] * t.DS[q * n + i] * t.DS[q * n + j];
      }
      t.M[i * n + j] = m;
      t.A[i * n + j] = a;
    }
  t.L = t.A;
  t.Nm.assign(n * n, 0);
  t.Np.assign(n * n, 0);
  const qr half = (qr)0.5;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      // face at xi = 0: nu = -1, own trace (v0, d0), neighbour trace at its xi = 1 (v1, d1)
      qr nu = -1;
      t.L[i * n + j] += sigma * t.v0[i] * t.v0[j] - half * nu * t.v0[i] * t.d0[j] - half * nu * t.d0[i] * t.v0[j];
      t.Nm[i * n + j] = -sigma * t.v0[i] * t.v1[j] - half * nu * t.v0[i] * t.d1[j] + half * nu * t.d0[i] * t.v1[j];
      // face at xi = 1: nu = +1, own (v1, d1), neighbour at its xi = 0 (v0, d0)
      nu = 1;
      t.L[i * n + j] += sigma * t.v1[i] * t.v1[j] - half * nu * t.v1[i] * t.d1[j] - half * nu * t.d1[i] * t.v1[j];
      t.Np[i * n + j] = -sigma * t.v1[i] * t.v0[j] - half * nu * t.v1[i] * t.d0[j] + half * nu * t.d1[i] * t.v0[j];
    }
  return t;
}

template <typename V>
void put(const V& src, double* dst) {
  for (size_t i = 0; i < src.size(); ++i) dst[i] = (double)src[i];
}

}  // namespace

bool build_tables(int p, int basis, double penalty_factor, Tables1D* out) {
  if (p < 1 || p + 1 > kMaxN || (basis != 0 && basis != 1)) return false;
  if (!(penalty_factor > 0)) penalty_factor = 1.0;
  const int n = p + 1;
  Tables1D& T = *out;
  T = Tables1D();
  T.p = p;
  T.n = n;
  T.basis = basis;
  std::vector<qr> xq, wq;
  gauss(n, xq, wq);
  put(xq, T.xq);
  put(wq, T.wq);
  qr sigma = (qr)(n * n) * (qr)penalty_factor;
  std::vector<QPoly> H = hermite_like(p);
  std::vector<QPoly> G = gl_lagrange(p);
  const std::vector<QPoly>& W = basis == 0 ? H : G;
  QTables q = build_q(W, xq, wq, sigma);
  put(q.S, T.S);
  put(q.DS, T.DS);
  put(q.v0, T.v0);
  put(q.v1, T.v1);
  put(q.d0, T.d0);
  put(q.d1, T.d1);
  put(q.M, T.Mhat);
  put(q.A, T.Ahat);
  put(q.L, T.Lhat);
  put(q.Nm, T.Nm);
  put(q.Np, T.Np);
  T.alpha1 = (double)q.d0[1];
  QTables g = build_q(G, xq, wq, sigma);
  put(g.M, T.gl_Mhat);
  put(g.L, T.gl_Lhat);
  put(g.Nm, T.gl_Nm);
  put(g.Np, T.gl_Np);
  put(g.S, T.gl_S);
  put(g.DS, T.gl_DS);
  put(g.v0, T.gl_v0);
  put(g.v1, T.gl_v1);
  put(g.d0, T.gl_d0);
  put(g.d1, T.gl_d1);
  // basis change: T[i][j] = phi_j^H(x_i^GL); identity when the working basis is GL
  std::vector<qr> Tm(n * n, 0);
  if (basis == 0) {
    std::vector<qr> xg = gl_points(n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) Tm[i * n + j] = H[j](xg[i]);
  } else {
    for (int i = 0; i < n; ++i) Tm[i * n + i] = 1;
  }
  put(Tm, T.T);
  put(inverse(Tm, n), T.Tinv);
  return true;
}

}  // namespace dgb
