// Internal host/device declarations of the dg_b200 library (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/dg.h"
#include "basis_host.h"
#include "common.cuh"

namespace dgb {

// Kernel parameters of the Cartesian Kronecker path (SURVEY.md §8(f) NEXT#1,
// Eq. (14)): per direction d, y = sum_d (Mhat (x) Mhat (x) L_d) u + neighbour
// couplings, L_d = (V/h_d^2) Lhat.  Passed by value (__grid_constant__), so all
// coefficients live in the constant bank.
template <typename Real>
struct KronParamsT {
  Real M[kEO];               // Mhat, even-odd packed, parity +1
  Real L[3][kEO];            // (V / h_d^2) Lhat, even-odd packed, parity +1
  Real Nm[3][kMaxN * kMaxN]; // [NL][NL]: own rows [0,NL) x neighbour layers [n-NL,n)
  Real Np[3][kMaxN * kMaxN]; // [NL][NL]: own rows [n-NL,n) x neighbour layers [0,NL)
  Real TiT[kEO];             // T^{-T}, even-odd packed
  Real Ti[kEO];              // T^{-1}
  // FDM block Jacobi (Eqs. (13)-(15)): L_hat Z = M_hat Z diag(lam), Z^T M_hat Z = I, split by
  // the reflection parity of the eigenvectors (hs symmetric, n - hs antisymmetric ones):
  //   Zs[i*hs + s] = Z[i][sym s]  for rows i < hs (row n/2 is the middle row for odd n)
  //   Za[i*ha + a] = Z[i][anti a] for rows i < n/2
  //   lam[m]: symmetric eigenvalues first, then antisymmetric (the packed eigen index)
  //   cdir[d] = V / h_d^2 (the direction weights of L_d)
  Real Zs[kMaxN * kMaxN];
  Real Za[kMaxN * kMaxN];
  Real lam[kMaxN];
  Real cdir[3];
  // Transformed-residual GL-Jacobi Chebyshev step (KMODE_CHEBY_GLT, NL = 2 only): the 1D
  // factors premultiplied by T^{-T}, so that the three matvec sweeps yield (T^{-T})^{(x)3} A u
  // directly (Kronecker mixed product); the rhs is transformed once per sweep.
  //   Mt = T^{-T} Mhat, Lt[d] = T^{-T} L_d (even-odd packed, parity +1)
  //   Ft[d]: P = T^{-T} N^-_d (n x NL, own rows x neighbour layers [n-NL, n)), even-odd packed
  //          with the mirror image T^{-T} N^+_d[n-1-i][NL-1-l] = P[i][l]:
  //          Fe[i][l] = (P[i][l] + P[n-1-i][l]) / 2, Fo[i][l] = (P[i][l] - P[n-1-i][l]) / 2
  //          (i < n/2), then Fm[l] = P[n/2][l] (odd n)
  Real Mt[kEO];
  Real Lt[3][kEO];
  Real Ft[3][kMaxN * 2];
};
using KronParams = KronParamsT<double>;
using KronParamsF = KronParamsT<float>;   // fp32 path, rounded from KronParams

// Where the z-neighbour layers of the bottom / top local plane come from.
enum { ZSRC_LOCAL = 0, ZSRC_HALO = 1, ZSRC_MIRROR = 2 };

struct GridArgs {
  int Nx, Ny, nz;             // local cells per direction (nz local planes)
  int bc[3];                  // DG_BC_* per direction (x, y used; z via zlo/zhi)
  int zlo, zhi;               // ZSRC_* for the plane below local plane 0 / above nz-1
  int zbeg, zend;             // local planes processed by this launch
  const double* halo_lo;      // [Nx*Ny][NL][n][n]: neighbour layers [n-NL, n) of the plane below
  const double* halo_hi;      // [Nx*Ny][NL][n][n]: neighbour layers [0, NL) of the plane above
  int l2pf;                   // k_kron4/k_quad: L2 prefetch of the next plane's tile (DG_L2PF, default 1)
};

enum { KMODE_APPLY = 0, KMODE_CHEBY_GL = 1, KMODE_CHEBY_PJ = 2, KMODE_CHEBY_FDM = 3,
       KMODE_CHEBY_GLT = 4 };   // GLT: GL-Jacobi step on the transformed residual (k_kron4, NL = 2)

template <typename Real>
struct ChebyArgsT {
  const Real* b;
  const Real* u_prev;         // may alias u_next (in-place three-term update)
  Real* u_next;
  const Real* dinv;           // inverse diagonal (GL for CHEBY_GL, working basis for CHEBY_PJ)
  double c_prev;              // rho_{j+1} rho_j      (0 on the first step)
  double c_z;                 // 2 rho_{j+1} / delta  (1/c on the first step)
  int first;                  // 1: u_prev is not read
};
using ChebyArgs = ChebyArgsT<double>;
using ChebyArgsF = ChebyArgsT<float>;

struct BchgParams {
  double B[kEO];              // even-odd packed 1D matrix, parity +1
};
struct BchgParamsF {
  float B[kEO];               // BchgParams rounded to float (fp32 path)
};

// Kernel parameters of the general quadrature path (Eqs. (3)-(5)):
// 1D tables in even-odd form, face traces restricted to the NL layers next to a
// face, and the constant-geometry data (DG_GEOM_CONSTANT).
struct QuadParams {
  double S[kEO];               // S[q][j] = phi_j(xq_q), parity +1
  double D[kEO];               // DS[q][j] = phi_j'(xq_q), parity -1
  double St[kEO];              // S^T
  double Dt[kEO];              // DS^T
  double sf[2][kMaxN];         // own trace  phi_L(s),  L = s ? n-NL+l : l
  double df[2][kMaxN];         // own trace  phi_L'(s)
  double sfn[2][kMaxN];        // neighbour trace phi_L(1-s), L = s ? l : n-NL+l
  double dfn[2][kMaxN];        // neighbour trace phi_L'(1-s)
  double w[kMaxN];             // Gauss weights on (0,1)
  double G0[6];                // CONSTANT: det J J^-1 J^-T  (xx, yy, zz, xy, xz, yz)
  double cw0[3][3];            // CONSTANT: det J |J^-T e_d| J^-1 n_+(d)   (times w_a w_b)
  double sdA0[3];              // CONSTANT: sigma_d det J |J^-T e_d|        (times w_a w_b)
  double TiT[kEO];             // T^{-T}
  double Ti[kEO];              // T^{-1}
};

enum { GEOM_CONST = 0, GEOM_PER_CELL = 1, GEOM_PER_QPOINT = 2 };

// Index of quadrature point (q0, q1, q2) (x, y, z) inside one [n^3] block of the per-q-point
// merged tensor: x slowest, then z, then y, so that the x-line threads (one per (q1, q2)) of
// the quadrature kernels read consecutive addresses at each position q0 along their line
// (coalesced 64-bit loads instead of per-thread runs of n).
template <int N>
__host__ __device__ __forceinline__ int gq(int q0, int q1, int q2) {
  return (q0 * N + q2) * N + q1;
}

// Geometry arrays of the general path (device pointers, library-owned).
struct GeomArgs {
  const double* G;             // PER_QPOINT: [cell][6][n^3 in gq order]  w_q det J J^-1 J^-T
  const double* face[3];       // PER_QPOINT: per direction [face][4][n^2]: dA J^-1 n_+ (3), sigma dA
  const double* jinv;          // PER_CELL:  [cell][10]: J^-1 (row-major), det J
  double pen;                  // (p+1)^2 * penalty_factor  (PER_CELL)
  const double* sig[3];        // PER_CELL with user penalties: sigma_F per face, layout of face[d]
};

// Analytic mesh map: x = L X + amp s(Xh), X = lo + (c+xi) h.
struct MapParams {
  double L[9];
  double h[3];
  double amp;
  int Nglob[3];
  int z0;                      // global index of local plane 0
  int bc[3];
  double pen;                  // (p+1)^2 * penalty_factor
  double xq[kMaxN], wq[kMaxN];
};

// Launchers (k_kron4.cu, k_kron6.cu, k_basis_change.cu, k_setup.cu)
// z-first Kronecker kernel (k_kron4.cu), the default Cartesian path for n = 3..9
bool kron4_supported(int n);
cudaError_t launch_kron4(int n, int NL, int mode, const KronParams& kp, const GridArgs& g,
                         const double* u, double* y, const ChebyArgs& ch, cudaStream_t s);
// n = 3 cell-per-thread Cartesian kernel (k_kron3c.cu): matvec and every fused Chebyshev mode
bool kron3c_supported(int n, int NL);
cudaError_t launch_kron3c(int NL, int mode, const KronParams& kp, const GridArgs& g, const double* u, double* y,
                          const ChebyArgs& ch, cudaStream_t s);
// i-plane Cartesian matvec (k_kron6.cu): z and y sweeps of a whole (j,k) plane per thread
bool kron6_supported(int n, int NL, int mode);
cudaError_t launch_kron6(int n, int mode, const KronParams& kp, const GridArgs& g, const double* u, double* y,
                         const ChebyArgs& ch, cudaStream_t s);
cudaError_t launch_kron4_f32(int n, int NL, int mode, const KronParamsF& kp, const GridArgs& g,
                             const float* u, float* y, const ChebyArgsF& ch, cudaStream_t s);
// z-first basis change (k_kron4.cu), n = 3..9; in == out is NOT allowed (z-lines are read
// while other blocks write)
cudaError_t launch_basis_change4(int n, const BchgParams& bp, const double* in, double* out, int64_t ncells,
                                 cudaStream_t s);
cudaError_t launch_basis_change(int n, const BchgParams& bp, const double* in, double* out,
                                int64_t ncells, cudaStream_t s);
cudaError_t launch_basis_change_f32(int n, const BchgParamsF& bp, const float* in, float* out,
                                    int64_t ncells, cudaStream_t s);
// warp-private pipelined basis change (k_bchgw.cu), in-place capable
cudaError_t launch_basis_change_w(int n, const BchgParams& bp, const double* in, double* out,
                                  int64_t ncells, cudaStream_t s);
cudaError_t launch_basis_change_w_f32(int n, const BchgParamsF& bp, const float* in, float* out,
                                      int64_t ncells, cudaStream_t s);
// diagonal of a Cartesian Kronecker operator: d[i,j,k] = sum_d c_d prod(1D diagonals)
struct CartDiagParams {
  double mdiag[kMaxN];                 // diag(Mhat_basis)
  double ldiag[3][4][kMaxN];           // per direction: [interior, left bdry, right bdry, both]
  double scale[3];                     // V / h_d^2
  int invert;                          // write 1/d instead of d
};
cudaError_t launch_cart_diag(int n, const CartDiagParams& p, int Nx, int Ny, int nz, int z0,
                             int Nz_global, double* out, cudaStream_t s);

cudaError_t measure_peak(int kind, double* value, cudaStream_t s);
cudaError_t launch_halo_pack(const double* u, double* send_lo, double* send_hi, int n, int NL,
                             int64_t plane_cells, int nz, cudaStream_t s);

// general quadrature path (k_quad.cu) and its setup (k_geom.cu)
cudaError_t launch_quad(int n, int NL, int geom, int mode, const QuadParams& qp, const GeomArgs& ga,
                        const GridArgs& g, const double* u, double* y, const ChebyArgs& ch,
                        cudaStream_t s);
// z-first quadrature kernel (k_quad3.cu): constant or per-q-point geometry, n = 3..9
bool quad3_supported(int n, int geom);
cudaError_t launch_quad3(int n, int NL, int geom, int mode, const QuadParams& qp, const GeomArgs& ga,
                         const GridArgs& g, const double* u, double* y, const ChebyArgs& ch,
                         cudaStream_t s);
// solver kernels (k_solver.cu): standalone P^{-1}, deterministic dot, vector updates
cudaError_t launch_pinv(int n, int inner, const KronParams& kp, const double* r, const double* dinv, double* z,
                        int64_t ncells, cudaStream_t s);
int dot_partials();
cudaError_t launch_d2f(const double* in, float* out, int64_t n, cudaStream_t s);
cudaError_t launch_f2d(const float* in, double* out, int64_t n, cudaStream_t s);
cudaError_t launch_dot(const double* a, const double* b, int64_t n, double* part, double* out, cudaStream_t s);
cudaError_t launch_axpby(double alpha, const double* x, double beta, double* y, int64_t n, cudaStream_t s);
cudaError_t launch_lanczos_start(double* v, int64_t n, int64_t g0, cudaStream_t s);
// usig[d] (may be NULL): the caller's sigma_F per face (dg.h user_penalty) replacing the
// computed mean; face layout of face[d]
cudaError_t launch_geom_qpoint(int n, const MapParams& mp, int Nx, int Ny, int nz, double* G,
                               double* face[3], const double* const usig[3], int* err_flag, cudaStream_t s);
// diagonal of the operator in a basis given by tables (S, DS, v0, v1, d0, d1 at the
// Gauss points), any geometry; invert -> 1/diag
struct DiagTables {
  double S[kMaxN * kMaxN], DS[kMaxN * kMaxN], v[2][kMaxN], d[2][kMaxN], w[kMaxN];
};
cudaError_t launch_diag_general(int n, int geom, const DiagTables& t, const QuadParams& qp,
                                const GeomArgs& ga, const GridArgs& g, int invert, double* out,
                                cudaStream_t s);

}  // namespace dgb
