// Host-side 1D tables for the CUDA kernels, built in __float128 and rounded to
// double (hard part (v): fp64 monomials drift at p=8).
#pragma once

namespace dgb {

constexpr int kMaxN = 9;   // n = p+1 <= 9

struct Tables1D {
  int p = 0, n = 0, basis = 0;
  double xq[kMaxN], wq[kMaxN];            // Gauss-Legendre points/weights on (0,1)
  double S[kMaxN * kMaxN];                // S[q*n+j]  = phi_j(xq_q)
  double DS[kMaxN * kMaxN];               // DS[q*n+j] = phi_j'(xq_q)
  double v0[kMaxN], v1[kMaxN];            // phi_j(0), phi_j(1)        (S_f)
  double d0[kMaxN], d1[kMaxN];            // phi_j'(0), phi_j'(1)      (D_f)
  // reference-interval 1D matrices (h = 1, sigma_hat = (p+1)^2 * penalty_factor)
  double Mhat[kMaxN * kMaxN];             // int phi_i phi_j
  double Ahat[kMaxN * kMaxN];             // int phi_i' phi_j'
  double Lhat[kMaxN * kMaxN];             // Ahat + own-side face terms at xi=0 and xi=1
  double Nm[kMaxN * kMaxN];               // own test (row) x neighbour trial (col), face xi=0
  double Np[kMaxN * kMaxN];               // own test (row) x neighbour trial (col), face xi=1
  double T[kMaxN * kMaxN];                // T[i*n+j] = phi_j^H(x_i^GL)   (identity for GL basis)
  double Tinv[kMaxN * kMaxN];
  // GL basis copies (for the GL-Jacobi diagonal of a Hermite mesh)
  double gl_Mhat[kMaxN * kMaxN], gl_Lhat[kMaxN * kMaxN], gl_Nm[kMaxN * kMaxN], gl_Np[kMaxN * kMaxN];
  double gl_S[kMaxN * kMaxN], gl_DS[kMaxN * kMaxN];
  double gl_v0[kMaxN], gl_v1[kMaxN], gl_d0[kMaxN], gl_d1[kMaxN];
  double alpha1 = 0;                      // D_f(0) = [-alpha1, alpha1, 0, ...] (Eq. (9))
};

// basis: 0 = Hermite-like, 1 = nodal Gauss-Lobatto.  Returns false on bad p.
bool build_tables(int p, int basis, double penalty_factor, Tables1D* out);

}  // namespace dgb
